"""Scenes and the density bake (fixture producers).

Mirrors of /root/reference/pkg/src/divas/scene.py:

* ``ScenePrimitive`` (scene.py:33-67, same validation), ``SceneModel``
  (scene.py:108-151) with the same ``packed()`` arrays;
* ``DensityGrid`` (scene.py:154-165);
* ``bake_density_grid`` (scene.py:194-201) -- one ``divas_bake_density``
  launch instead of a per-primitive numpy pass (and, when unbounded, a
  Python loop of ``contract`` per voxel centre).  Bit-identical to the
  reference (tests/test_render_golden.py, tests/test_gpu_render.py).

The hot-path functions accept the reference's own scene objects too: they
only call ``packed()`` and read ``background`` / ``bounds``.
"""

from __future__ import annotations

import ctypes
from dataclasses import dataclass

import numpy as np

from . import _native
from ._device import device, empty
from .geometry import SceneBounds, VoxelGrid

__all__ = ["ScenePrimitive", "SceneModel", "DensityGrid", "bake_density_grid",
           "bake_density_device"]

KIND_SPHERE, KIND_BOX, KIND_CAPSULE = 0, 1, 2
_KIND_NAMES = {"sphere": KIND_SPHERE, "box": KIND_BOX, "capsule": KIND_CAPSULE}


@dataclass(frozen=True)
class ScenePrimitive:
    """sphere {center, radius, inner_radius=0} | box {center, half_extents} |
    capsule {p0, p1, radius}; density, color, object_id >= 1, soft_edge >= 0."""

    kind: str
    params: dict
    density: float
    color: tuple
    object_id: int
    soft_edge: float = 0.0

    def __post_init__(self):                       # scene.py:49-67
        if self.kind not in _KIND_NAMES:
            raise ValueError(f"unknown primitive kind {self.kind!r}")
        if self.density < 0:
            raise ValueError("density must be >= 0")
        if self.soft_edge < 0:
            raise ValueError("soft edge width must be >= 0")
        if self.object_id < 1:
            raise ValueError("object ids start at 1")
        if self.kind == "sphere":
            if self.params["radius"] <= 0:
                raise ValueError("sphere radius must be positive")
            inner = self.params.get("inner_radius", 0.0)
            if inner < 0 or inner >= self.params["radius"]:
                raise ValueError("inner radius must lie in [0, radius)")
        if self.kind == "box" and np.any(np.asarray(self.params["half_extents"]) <= 0):
            raise ValueError("box half extents must be positive")
        if self.kind == "capsule" and self.params["radius"] <= 0:
            raise ValueError("capsule radius must be positive")


@dataclass(frozen=True)
class SceneModel:
    primitives: tuple
    bounds: SceneBounds
    background: tuple = (0.0, 0.0, 0.0)

    def __post_init__(self):
        object.__setattr__(self, "primitives", tuple(self.primitives))
        object.__setattr__(self, "background", tuple(float(c) for c in self.background))

    def object_ids(self):
        return sorted({p.object_id for p in self.primitives})

    def packed(self):
        """(kinds u8, params (N,7) f64, densities f64, colors (N,3) f64,
        object_ids i32, soft_edges f64) -- scene.py:126-151's layout."""
        n = len(self.primitives)
        kinds = np.zeros(n, dtype=np.uint8)
        params = np.zeros((n, 7), dtype=np.float64)
        dens = np.zeros(n, dtype=np.float64)
        cols = np.zeros((n, 3), dtype=np.float64)
        oids = np.zeros(n, dtype=np.int32)
        soft = np.zeros(n, dtype=np.float64)
        for i, pr in enumerate(self.primitives):
            kinds[i] = _KIND_NAMES[pr.kind]
            if pr.kind == "sphere":
                params[i, :3] = pr.params["center"]
                params[i, 3] = pr.params["radius"]
                params[i, 4] = pr.params.get("inner_radius", 0.0)
            elif pr.kind == "box":
                params[i, :3] = pr.params["center"]
                params[i, 3:6] = pr.params["half_extents"]
            else:
                params[i, :3] = pr.params["p0"]
                params[i, 3:6] = pr.params["p1"]
                params[i, 6] = pr.params["radius"]
            dens[i] = pr.density
            cols[i] = pr.color
            oids[i] = pr.object_id
            soft[i] = pr.soft_edge
        return kinds, params, dens, cols, oids, soft


@dataclass
class DensityGrid:
    grid: VoxelGrid
    values: np.ndarray  # (G, G, G) float32, indexed [ix, iy, iz]

    def __post_init__(self):
        g = self.grid.resolution
        self.values = np.asarray(self.values, dtype=np.float32).reshape(g, g, g)
        if not np.all(np.isfinite(self.values)) or np.any(self.values < 0):
            raise ValueError("densities must be finite and >= 0")


def scene_struct(scene):
    """(``divas_scene`` struct, keep-alive arrays) of a SceneModel-like object."""
    kinds, params, dens, cols, _oids, soft = scene.packed()
    keep = [np.ascontiguousarray(kinds, np.uint8), np.ascontiguousarray(params, np.float64),
            np.ascontiguousarray(dens, np.float64), np.ascontiguousarray(cols, np.float64),
            np.ascontiguousarray(soft, np.float64)]
    n = len(keep[0])
    if n > _native.MAX_PRIMS:
        raise ValueError(f"{n} primitives: the device marcher takes up to {_native.MAX_PRIMS}")
    st = _native.Scene()
    st.n_prims = n
    st.kinds, st.params, st.density, st.colors, st.soft = (a.ctypes.data for a in keep)
    st.background = (ctypes.c_double * 3)(*[float(c) for c in scene.background])
    return st, keep


def bake_density_device(scene, grid, dev=None, stream=None):
    """``bake_density_grid`` values as a CUDA f32 tensor (G, G, G)."""
    dev = dev or device()
    st, _keep = scene_struct(scene)
    g = int(grid.resolution)
    out = empty((g, g, g), np.float32, dev)
    b = scene.bounds
    unb = 1 if getattr(b, "unbounded", False) else 0
    lo, hi = np.asarray(b.min, np.float64), np.asarray(b.max, np.float64)
    bc, bh = 0.5 * (lo + hi), 0.5 * (hi - lo)               # SceneBounds.center / half
    D3 = ctypes.c_double * 3
    _native.check(_native.lib().divas_bake_density(
        ctypes.byref(st), g, D3(*np.asarray(grid.origin, np.float64).reshape(3)),
        float(grid.voxel_size()), unb, D3(*bc), D3(*bh), _native.ptr(out),
        _native.stream_handle(stream)), "bake_density_grid")
    return out


def bake_density_grid(scene, grid) -> DensityGrid:
    """Sample scene density at voxel centers (contracted when unbounded)."""
    out = bake_density_device(scene, grid)
    return DensityGrid(grid, out.cpu().numpy())
