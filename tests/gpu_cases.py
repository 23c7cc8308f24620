"""Helpers that turn golden cases into device inputs / reference-style objects."""

import types

import numpy as np

from paper_2601_04860_b200.geometry import Camera, SceneBounds, VoxelGrid
from paper_2601_04860_b200.render import ViewGeometry
from paper_2601_04860_b200.scene import DensityGrid
from paper_2601_04860_b200.segmenter import ConfidenceMask


def cams_array(case):
    nv = case.rots.shape[0]
    return np.concatenate([case.rots.reshape(nv, 9), case.poss, case.intr], axis=1)


def device_views(case, dev, perm=None):
    import torch
    from paper_2601_04860_b200.fusion import DeviceViews
    order = np.arange(case.rots.shape[0]) if perm is None else np.asarray(perm)
    t = lambda a: torch.from_numpy(np.ascontiguousarray(a[order])).to(dev)  # noqa: E731
    return DeviceViews(t(cams_array(case)), t(case.masks), t(case.dmins), t(case.dmaxs),
                       t(case.dexps), t(case.nsamps))


def grid_ns(case):
    return types.SimpleNamespace(resolution=case.g, origin=case.origin,
                                 voxel_size=lambda: case.dx)


def bounds_ns(case):
    if not case.unb:
        return None
    return types.SimpleNamespace(unbounded=True, center=case.bc, half=case.bh)


def reference_objects(case):
    """(VoxelGrid, DensityGrid, views, bounds) in the reference's object model."""
    grid = VoxelGrid(case.g, case.half, case.origin)
    assert grid.voxel_size() == case.dx
    dens = DensityGrid(grid, case.density.reshape(case.g, case.g, case.g))
    views = []
    for i in range(case.rots.shape[0]):
        fx, fy, cx, cy, w, h = case.intr[i]
        w, h = int(w), int(h)
        m4 = np.eye(4)
        m4[:3, :3] = case.rots[i]
        m4[:3, 3] = case.poss[i]
        cam = Camera(fx=fx, fy=fy, cx=cx, cy=cy, width=w, height=h, world_from_camera=m4)
        sl = np.s_[i, :h, :w]
        vg = ViewGeometry(cam, np.zeros((h, w, 3), np.float32), case.dmins[sl].copy(),
                          case.dmaxs[sl].copy(), case.dexps[sl].copy(), case.nsamps[sl].copy(),
                          case.dexps[sl].copy())
        views.append((vg, ConfidenceMask(case.masks[sl].copy(), refined=True)))
    bounds = None
    if case.unb:
        bounds = SceneBounds(case.bc - case.bh, case.bc + case.bh, unbounded=True)
    return grid, dens, views, bounds
