"""Incremental, device-resident session fusion (BASELINE config C4).

The reference session re-packs, re-grades and re-fuses every mask on every
update (`Session.maybe_fuse`, /root/reference/pkg/src/divas/session.py:189-230;
"each fusion is a full recompute", `:212-215`).  Here the state of a fusion
stays in HBM between updates:

* view planes, cameras and the per-view aux (scan records + depth bands) for
  up to ``max_views`` views;
* the fusion workspace: the density-gated voxel list and every (view, voxel)
  contribution (w, m*w / t) with its presence bit;
* the outputs p and occupancy.

Adding a view, or replacing (re-refining) one view's mask, refines that view
alone, re-evaluates only its (view, voxel) pairs (`divas_fuse` in
INCREMENTAL mode clears the view's bits, runs the pair kernel for it, then
re-runs the value-sorted reduction over all views).  Because the per-voxel
sums are taken in value-sorted order, the result is bit-identical to a full
`fuse` of the current view set (tests/test_gpu_incremental.py).
"""

from __future__ import annotations

import numpy as np

from . import _native
from ._device import as_device, device
from .fusion import (DeviceViews, Fuser, OccupancyGrid, _check_layout, _sparse_probs_to_host,
                     pack_cameras)
from .segmenter import ViewAux, refine_bands_device

__all__ = ["FusionSession"]


class FusionSession:
    """Device-resident fusion state for one grid, density and parameter set.

    ``shape`` is the (height, width) of the largest view the session will
    hold; ``max_views`` bounds the view count (workspace sizing).
    """

    def __init__(self, grid, density, params, shape, bounds=None, max_views=64, dev=None):
        import torch
        _check_layout(grid, density)
        self.grid = grid
        self.g = int(grid.resolution)
        self.dev = dev or device()
        self.hm, self.wm = int(shape[0]), int(shape[1])
        self.max_views = int(max_views)
        self.fuser = Fuser(grid, params, bounds)
        self.density = as_device(density.values, np.float32, self.dev).reshape(-1)
        shp = (self.max_views, self.hm, self.wm)
        z = lambda dt: torch.zeros(shp, dtype=dt, device=self.dev)  # noqa: E731
        self.raw, self.z = z(torch.float32), z(torch.float32)
        self.dmins, self.dmaxs, self.dexps = z(torch.float32), z(torch.float32), z(torch.float32)
        self.nsamps = z(torch.int32)
        self.cams = torch.zeros((self.max_views, _native.CAM_STRIDE), dtype=torch.float64,
                                device=self.dev)
        self.aux = ViewAux.empty(self.max_views, self.hm, self.wm, self.dev)
        self.probs = torch.zeros(self.g ** 3, dtype=torch.float64, device=self.dev)
        self.occ = torch.zeros(self.g ** 3, dtype=torch.uint8, device=self.dev)
        self.sizes = []
        self.nv = 0
        self._ws = None
        self._cap = self.fuser.capacity(self.density, 0, self.g ** 3)
        self._fused = False
        self._out = None
        self._graphs = {}          # (view, nv) -> CUDA graph of its re-refine + re-fuse
        self._rois = None          # per-view record windows (sharding.slab_view_rois)

    # -- state ---------------------------------------------------------------
    def _views(self):
        n = self.nv
        return DeviceViews(self.cams[:n], self.raw[:n], self.dmins[:n], self.dmaxs[:n],
                           self.dexps[:n], self.nsamps[:n], sizes=self.sizes)

    def _upload(self, i, view, mask):
        import torch
        cam = view.camera
        h, w = int(cam.height), int(cam.width)
        mv = mask.values if hasattr(mask, "values") else np.asarray(mask)
        if getattr(mask, "refined", False):
            raise ValueError("mask is already refined")
        if tuple(mv.shape) != (h, w) or tuple(view.z_surface.shape) != (h, w):
            raise ValueError("mask and view dimensions differ")
        if h > self.hm or w > self.wm:
            raise ValueError(f"view {h}x{w} exceeds the session's {self.hm}x{self.wm} planes")
        src = {"raw": mv, "z": view.z_surface, "dmins": view.d_min, "dmaxs": view.d_max,
               "dexps": view.d_exp, "nsamps": view.n_samples}
        for k, arr in src.items():
            plane = getattr(self, k)[i]
            dt = np.int32 if k == "nsamps" else np.float32
            if (h, w) != (self.hm, self.wm):
                plane.zero_()
            plane[:h, :w].copy_(torch.from_numpy(np.ascontiguousarray(arr, dt)))
        self.cams[i].copy_(torch.from_numpy(pack_cameras([cam])[0]))
        self._rois = None          # new camera: new windows (and captured graphs use the old)
        self._graphs.clear()
        if i == len(self.sizes):
            self.sizes.append((h, w))
        else:
            self.sizes[i] = (h, w)

    def _windows(self):
        """The views' record windows: the fusion reads no record or band
        outside the projection of the gated voxels' bounding box (DESIGN.md
        section 3), so a view's refine + band pass runs only there.  Fixed by
        the density and the cameras; recomputed when the view set changes."""
        if self._rois is None or self._rois.nv != self.nv:
            from .sharding import slab_view_rois
            self._rois = slab_view_rois(self.density, self.fuser.pv, self.g,
                                        self.fuser.origin, self.fuser.dx,
                                        self.cams[:self.nv].cpu().numpy(), self.sizes)
        return self._rois

    def _refine(self, v0, v1):
        recs, bands = self.aux.view_slices(v0, v1, self.max_views, self.hm, self.wm)
        refine_bands_device(self.raw[v0:v1], self.z[v0:v1], self.nsamps[v0:v1],
                            self.dexps[v0:v1], self.fuser.pv, self.fuser.dx,
                            aux=(recs, bands), planar=False,
                            roi=self._windows().subset(v0, v1))

    def _fuse(self, v0, v1):
        incr = (v0, v1) if self._fused else None
        out = self.fuser.run(self.density, self._views(), probs=self.probs, occ=self.occ,
                             workspace=self._ws, max_gated=self._cap, aux=self.aux,
                             nv_cap=self.max_views, incremental=incr)
        self._ws = out["workspace"]
        self._out = out
        self._fused = True

    # -- updates (all asynchronous on the current stream) ----------------------
    def add_views(self, pairs):
        """Append (ViewGeometry, raw ConfidenceMask) pairs; refine and fuse them."""
        pairs = list(pairs)
        if not pairs:
            return
        if self.nv + len(pairs) > self.max_views:
            raise ValueError("session view capacity exceeded")
        v0 = self.nv
        for k, (vg, m) in enumerate(pairs):
            self._upload(v0 + k, vg, m)
        self.nv += len(pairs)
        self._graphs.clear()       # captured launches carry the old view count
        self._refine(v0, self.nv)
        self._fuse(v0, self.nv)

    def add_view(self, view, raw_mask) -> int:
        self.add_views([(view, raw_mask)])
        return self.nv - 1

    def replace_mask(self, index, raw_mask, view=None):
        """New raw mask (and optionally new maps) for view ``index``: re-refine
        and re-fuse that view only."""
        if not 0 <= index < self.nv:
            raise IndexError(index)
        if view is None:
            import torch
            h, w = self.sizes[index]
            mv = raw_mask.values if hasattr(raw_mask, "values") else np.asarray(raw_mask)
            if getattr(raw_mask, "refined", False):
                raise ValueError("mask is already refined")
            if tuple(mv.shape) != (h, w):
                raise ValueError("mask and view dimensions differ")
            self.raw[index, :h, :w].copy_(torch.from_numpy(np.ascontiguousarray(mv, np.float32)))
        else:
            self._upload(index, view, raw_mask)
        self._refine(index, index + 1)
        self._fuse(index, index + 1)

    def replace_mask_device(self, index, raw_plane, graph=True):
        """As ``replace_mask`` with the new raw mask already on the device
        (a [h, w] float32 CUDA tensor); no host synchronisation.

        ``graph``: the view's re-refine + re-fuse launches (refine init /
        min-max / band pass, clear bits, pair kernel, reduction) are captured
        once into a CUDA graph and replayed, so an update costs one graph
        launch instead of the Python / driver overhead of six kernel launches.
        """
        import torch
        if not 0 <= index < self.nv:
            raise IndexError(index)
        h, w = self.sizes[index]
        if tuple(raw_plane.shape) != (h, w):
            raise ValueError("mask and view dimensions differ")
        self.raw[index, :h, :w].copy_(raw_plane)
        if not (graph and self._fused):
            self._refine(index, index + 1)
            self._fuse(index, index + 1)
            return
        key = (index, self.nv)
        g = self._graphs.get(key)
        if g is None:
            g = torch.cuda.CUDAGraph()
            side = torch.cuda.Stream(device=self.dev)
            side.wait_stream(torch.cuda.current_stream(self.dev))
            with torch.cuda.stream(side):             # warm the allocator outside capture
                self._refine(index, index + 1)
                self._fuse(index, index + 1)
            torch.cuda.current_stream(self.dev).wait_stream(side)
            with torch.cuda.graph(g):
                self._refine(index, index + 1)
                self._fuse(index, index + 1)
            self._graphs[key] = g
        g.replay()

    def pop_view(self):
        """Drop the last view: its contribution bits are cleared and the
        value-sorted sums re-taken over the remaining views (bit-identical to
        a fusion of the remaining view set)."""
        if self.nv == 0:
            raise IndexError("the session holds no view")
        i = self.nv - 1
        if self._fused:
            out = self.fuser.run(self.density, self._views(), probs=self.probs, occ=self.occ,
                                 workspace=self._ws, max_gated=self._cap, aux=self.aux,
                                 nv_cap=self.max_views, view_range=(i, i + 1),
                                 steps=_native.STEP_CLEAR_VIEWS | _native.STEP_REDUCE)
            self._ws = out["workspace"]
            self._out = out
        self.nv -= 1
        self.sizes.pop()
        self._graphs.clear()
        self._rois = None

    def refuse(self):
        """Full recompute of the current view set (same result, for checking)."""
        self._fused = False
        self._fuse(0, self.nv)

    # -- results ---------------------------------------------------------------
    def occupancy_grid(self) -> OccupancyGrid:
        """Host OccupancyGrid of the current state (syncs)."""
        if self._out is None:
            return OccupancyGrid(self.grid, np.zeros((self.g,) * 3))
        return OccupancyGrid(self.grid, _sparse_probs_to_host(self._out, self.g ** 3)
                             .reshape((self.g,) * 3))
