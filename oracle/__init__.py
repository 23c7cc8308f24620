"""CPU oracle for the DivAS fusion hot path -- TEST INFRASTRUCTURE ONLY.

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py`` (its
``cpu_baseline`` leg and ``--impl reference``) may import this module, and
only as the checker / CPU baseline.  The product package
``paper_2601_04860_b200`` never imports it and has no CPU fallback.

The arithmetic lives in ``divas_oracle.c`` (a plain-C restatement of the
reference's numba kernels, built with ``-ffp-contract=off``); this module is
the numpy-facing wrapper plus the host-side packing, which restates the
reference's ``_pack_views`` (``/root/reference/pkg/src/divas/fusion.py:653-681``)
and ``FusionParams.as_vector`` (``fusion.py:80-87``).

Parity is pinned: ``tests/test_oracle_golden.py`` checks every function here
bit-for-bit against golden vectors that the reference itself produced
(``tests/golden/make_golden.py``).
"""

from __future__ import annotations

import ctypes
import os
import subprocess
import threading

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_LIB_PATH = os.path.join(_HERE, "_build", "liboracle.so")
_lib = None
_lock = threading.Lock()

_F32P = ctypes.POINTER(ctypes.c_float)
_F64P = ctypes.POINTER(ctypes.c_double)
_I32P = ctypes.POINTER(ctypes.c_int32)
_U8P = ctypes.POINTER(ctypes.c_uint8)


class _FuseArgs(ctypes.Structure):
    _fields_ = [
        ("g", ctypes.c_int64), ("origin", _F64P), ("dx_vox", ctypes.c_double),
        ("density", _F32P), ("nv", ctypes.c_int64), ("hm", ctypes.c_int64),
        ("wm", ctypes.c_int64), ("rots", _F64P), ("poss", _F64P), ("intr", _F64P),
        ("masks", _F32P), ("dmins", _F32P), ("dmaxs", _F32P), ("dexps", _F32P),
        ("nsamps", _I32P), ("valids", _U8P), ("gmaps", _F64P), ("pv", _F64P),
        ("bc", _F64P), ("bh", _F64P), ("unbounded", ctypes.c_int64),
        ("vox_lo", ctypes.c_int64), ("vox_hi", ctypes.c_int64),
        ("early_out", ctypes.c_int64), ("nthreads", ctypes.c_int64),
        ("out", _F64P), ("n_thick", _I32P), ("n_thin", _I32P),
        ("sw", _F64P), ("smw", _F64P), ("st", _F64P),
    ]


class _Scene(ctypes.Structure):
    _fields_ = [("n", ctypes.c_int64), ("kinds", _U8P), ("params", _F64P), ("dens", _F64P),
                ("cols", _F64P), ("soft", _F64P), ("bg", _F64P)]


class _RenderCfg(ctypes.Structure):
    _fields_ = [("n_steps", ctypes.c_int64), ("near_", ctypes.c_double),
                ("far_", ctypes.c_double), ("tau_cw", ctypes.c_double),
                ("min_w", ctypes.c_double)]


def build(force: bool = False) -> str:
    """Compile divas_oracle.c with the committed Makefile; returns the .so path."""
    srcs = ("divas_oracle.c", "divas_oracle_render.c", "Makefile")
    if force or not os.path.exists(_LIB_PATH) or os.path.getmtime(_LIB_PATH) < max(
            os.path.getmtime(os.path.join(_HERE, f)) for f in srcs):
        subprocess.run(["make", "-s", "-C", _HERE], check=True)
    return _LIB_PATH


def load():
    global _lib
    with _lock:
        if _lib is None:
            build()
            lib = ctypes.CDLL(_LIB_PATH)
            lib.oracle_refine.argtypes = [ctypes.c_int64, ctypes.c_int64, _F32P, _F32P, _I32P, _F32P]
            lib.oracle_gradient_maps.argtypes = [ctypes.c_int64] * 3 + [_F32P, _F32P, _F32P, _U8P,
                                                                       ctypes.c_double, ctypes.c_double, _F64P]
            lib.oracle_fuse.argtypes = [ctypes.POINTER(_FuseArgs)]
            lib.oracle_max_threads.restype = ctypes.c_int
            sp, rp = ctypes.POINTER(_Scene), ctypes.POINTER(_RenderCfg)
            lib.oracle_march.argtypes = [sp, rp, _F64P, _F64P]
            lib.oracle_render.argtypes = [sp, rp, _F64P, _F64P, _F64P, _F32P, _F32P, _F32P,
                                          _F32P, _I32P, _F32P, ctypes.c_int64]
            lib.oracle_bake.argtypes = [sp, ctypes.c_int64, _F64P, ctypes.c_double,
                                        ctypes.c_int64, _F64P, _F64P, _F32P, ctypes.c_int64]
            _lib = lib
    return _lib


def max_threads() -> int:
    return int(load().oracle_max_threads())


def _p(a, t):
    return a.ctypes.data_as(t) if a is not None else ctypes.cast(None, t)


def _c(a, dtype):
    return np.ascontiguousarray(a, dtype=dtype)


# --------------------------------------------------------------------------
# refine_mask (segmenter.py:129-152)
# --------------------------------------------------------------------------

def refine(mask, z_surface, n_samples) -> np.ndarray:
    """Depth-weighted refinement of one (H, W) mask; returns float32 (H, W)."""
    m = _c(mask, np.float32)
    z = _c(z_surface, np.float32)
    n = _c(n_samples, np.int32)
    if m.shape != z.shape or m.shape != n.shape or m.ndim != 2:
        raise ValueError("mask and view dimensions differ")
    out = np.empty_like(m)
    load().oracle_refine(m.shape[0], m.shape[1], _p(m, _F32P), _p(z, _F32P), _p(n, _I32P), _p(out, _F32P))
    return out


# --------------------------------------------------------------------------
# packing (fusion.py:653-681) and gradient maps (fusion.py:684-689)
# --------------------------------------------------------------------------

def _mask_values(m):
    return m.values if hasattr(m, "values") else np.asarray(m)


def pack_views(views):
    """Restates `_pack_views`: pad every view to (Hmax, Wmax), SoA arrays."""
    cams = [vg.camera for vg, _m in views]
    hmax = max(int(c.height) for c in cams)
    wmax = max(int(c.width) for c in cams)
    nv = len(views)
    rots = np.zeros((nv, 3, 3))
    poss = np.zeros((nv, 3))
    intr = np.zeros((nv, 6))
    masks = np.zeros((nv, hmax, wmax), dtype=np.float32)
    dmins = np.zeros((nv, hmax, wmax), dtype=np.float32)
    dmaxs = np.zeros((nv, hmax, wmax), dtype=np.float32)
    dexps = np.zeros((nv, hmax, wmax), dtype=np.float32)
    nsamps = np.zeros((nv, hmax, wmax), dtype=np.int32)
    valids = np.zeros((nv, hmax, wmax), dtype=np.uint8)
    for i, (vg, m) in enumerate(views):
        c = vg.camera
        mv = _mask_values(m)
        if mv.shape != (c.height, c.width):
            raise ValueError("mask and view dimensions differ")
        rots[i] = c.rotation
        poss[i] = c.position
        intr[i] = (c.fx, c.fy, c.cx, c.cy, float(c.width), float(c.height))
        sl = np.s_[i, :c.height, :c.width]
        masks[sl] = mv
        dmins[sl] = vg.d_min
        dmaxs[sl] = vg.d_max
        dexps[sl] = vg.d_exp
        nsamps[sl] = vg.n_samples
        valids[sl] = np.asarray(vg.n_samples) > 0
    return rots, poss, intr, masks, dmins, dmaxs, dexps, nsamps, valids


def gradient_maps(dexps, dmins, dmaxs, valids, eps, kappa) -> np.ndarray:
    dexps = _c(dexps, np.float32)
    dmins = _c(dmins, np.float32)
    dmaxs = _c(dmaxs, np.float32)
    valids = _c(valids, np.uint8)
    nv, h, w = dexps.shape
    out = np.zeros((nv, h, w), dtype=np.float64)
    load().oracle_gradient_maps(nv, h, w, _p(dexps, _F32P), _p(dmins, _F32P), _p(dmaxs, _F32P),
                                _p(valids, _U8P), float(eps), float(kappa), _p(out, _F64P))
    return out


def params_vector(params) -> np.ndarray:
    """FusionParams.as_vector() (fusion.py:80-87); accepts an array as-is."""
    if hasattr(params, "as_vector"):
        return np.asarray(params.as_vector(), dtype=np.float64)
    pv = np.asarray(params, dtype=np.float64)
    if pv.shape != (14,):
        raise ValueError("params vector must have 14 entries")
    return pv


def bounds_arrays(bounds):
    """fusion.py:542-546."""
    if bounds is None or not bounds.unbounded:
        return np.zeros(3), np.ones(3), 0
    return (np.ascontiguousarray(bounds.center, dtype=np.float64),
            np.ascontiguousarray(bounds.half, dtype=np.float64), 1)


# --------------------------------------------------------------------------
# fusion (fusion.py:692-724, kernel :410-509)
# --------------------------------------------------------------------------

def fuse_packed(g, origin, dx_vox, density, packed, pv, bc, bh, unbounded,
                gmaps=None, vox_range=None, early_out=True, nthreads=0,
                stats=True):
    """Run the oracle kernel on packed arrays.

    Returns a dict with ``p`` (G^3 f64) and, if ``stats``, the integer votes
    ``n_thick``/``n_thin`` and sorted sums ``sw``/``smw``/``st``.
    Voxels outside ``vox_range`` are left at zero.
    """
    rots, poss, intr, masks, dmins, dmaxs, dexps, nsamps, valids = packed
    rots = _c(rots, np.float64)
    poss = _c(poss, np.float64)
    intr = _c(intr, np.float64)
    masks = _c(masks, np.float32)
    dmins = _c(dmins, np.float32)
    dmaxs = _c(dmaxs, np.float32)
    dexps = _c(dexps, np.float32)
    nsamps = _c(nsamps, np.int32)
    valids = _c(valids, np.uint8)
    pv = _c(params_vector(pv), np.float64)
    if gmaps is None:
        gmaps = gradient_maps(dexps, dmins, dmaxs, valids, pv[9], pv[12])
    gmaps = _c(gmaps, np.float64)
    dens = _c(density, np.float32).reshape(-1)
    nvox = int(g) ** 3
    if dens.size != nvox:
        raise ValueError("density grid layout does not match the fusion grid")
    origin = _c(origin, np.float64).reshape(3)
    bc = _c(bc, np.float64).reshape(3)
    bh = _c(bh, np.float64).reshape(3)
    lo, hi = (0, nvox) if vox_range is None else (int(vox_range[0]), int(vox_range[1]))
    out = np.zeros(nvox, dtype=np.float64)
    res = {"p": out}
    if stats:
        for k in ("n_thick", "n_thin"):
            res[k] = np.zeros(nvox, dtype=np.int32)
        for k in ("sw", "smw", "st"):
            res[k] = np.zeros(nvox, dtype=np.float64)
    nv, hm, wm = masks.shape
    a = _FuseArgs(
        g=int(g), origin=_p(origin, _F64P), dx_vox=float(dx_vox), density=_p(dens, _F32P),
        nv=nv, hm=hm, wm=wm, rots=_p(rots, _F64P), poss=_p(poss, _F64P), intr=_p(intr, _F64P),
        masks=_p(masks, _F32P), dmins=_p(dmins, _F32P), dmaxs=_p(dmaxs, _F32P),
        dexps=_p(dexps, _F32P), nsamps=_p(nsamps, _I32P), valids=_p(valids, _U8P),
        gmaps=_p(gmaps, _F64P), pv=_p(pv, _F64P), bc=_p(bc, _F64P), bh=_p(bh, _F64P),
        unbounded=int(unbounded), vox_lo=lo, vox_hi=hi, early_out=1 if early_out else 0,
        nthreads=int(nthreads), out=_p(out, _F64P),
        n_thick=_p(res.get("n_thick"), _I32P), n_thin=_p(res.get("n_thin"), _I32P),
        sw=_p(res.get("sw"), _F64P), smw=_p(res.get("smw"), _F64P), st=_p(res.get("st"), _F64P),
    )
    load().oracle_fuse(ctypes.byref(a))
    return res


def fuse(grid, density, views, params, bounds=None, early_out=True, nthreads=0,
         stats=True):
    """Oracle twin of ``divas.fusion.fuse`` on duck-typed reference objects.

    ``grid`` has ``resolution``, ``origin``, ``voxel_size()``; ``density`` has
    ``values`` (G,G,G) f32; ``views`` is a list of (ViewGeometry, mask) pairs.
    Returns the dict of ``fuse_packed`` with ``p`` reshaped to (G,G,G).
    """
    g = int(grid.resolution)
    dvals = density.values if hasattr(density, "values") else density
    if not views:
        z = {"p": np.zeros((g, g, g))}
        if stats:
            z.update(n_thick=np.zeros(g ** 3, np.int32), n_thin=np.zeros(g ** 3, np.int32),
                     sw=np.zeros(g ** 3), smw=np.zeros(g ** 3), st=np.zeros(g ** 3))
        return z
    packed = pack_views(views)
    bc, bh, unb = bounds_arrays(bounds)
    res = fuse_packed(g, grid.origin, grid.voxel_size(), dvals, packed, params_vector(params),
                      bc, bh, unb, early_out=early_out, nthreads=nthreads, stats=stats)
    res["p"] = res["p"].reshape(g, g, g)
    return res


# --------------------------------------------------------------------------
# threshold / extract (ablation.py:109, np.argwhere C-order)
# --------------------------------------------------------------------------

def threshold(probs, thr=0.5) -> np.ndarray:
    return np.asarray(probs) >= thr


def extract(probs, thr=0.5) -> np.ndarray:
    return np.argwhere(np.asarray(probs) >= thr)


# --------------------------------------------------------------------------
# fixture producers: render_view / march_ray (render.py:96-292) and
# bake_density_grid (scene.py:194-201)
# --------------------------------------------------------------------------

def _scene_struct(scene):
    """(ctypes struct, keep-alive arrays) from a SceneModel-like object
    (``.packed()`` + ``.background``) or a packed tuple
    (kinds, params, dens, cols, soft, bg)."""
    if hasattr(scene, "packed"):
        kinds, params, dens, cols, _oids, soft = scene.packed()
        bg = scene.background
    else:
        kinds, params, dens, cols, soft, bg = scene
    keep = [_c(kinds, np.uint8).reshape(-1), _c(params, np.float64).reshape(-1, 7),
            _c(dens, np.float64).reshape(-1), _c(cols, np.float64).reshape(-1, 3),
            _c(soft, np.float64).reshape(-1), _c(bg, np.float64).reshape(3)]
    st = _Scene(len(keep[0]), _p(keep[0], _U8P), _p(keep[1], _F64P), _p(keep[2], _F64P),
                _p(keep[3], _F64P), _p(keep[4], _F64P), _p(keep[5], _F64P))
    return st, keep


def _cfg_struct(cfg):
    if hasattr(cfg, "samples_per_ray"):
        cfg = (cfg.samples_per_ray, cfg.near, cfg.far, cfg.tau_cw, cfg.min_weight)
    return _RenderCfg(int(cfg[0]), float(cfg[1]), float(cfg[2]), float(cfg[3]), float(cfg[4]))


def march(scene, cfg, rays) -> np.ndarray:
    """``_march`` on unit rays (n, 6) = origin, direction; returns (n, 8) f64
    (r, g, b, d_min, d_max, d_exp, n_samples, z_surface)."""
    st, _keep = _scene_struct(scene)
    rc = _cfg_struct(cfg)
    rays = _c(rays, np.float64).reshape(-1, 6)
    out = np.zeros((len(rays), 8))
    lib = load()
    for i in range(len(rays)):
        lib.oracle_march(ctypes.byref(st), ctypes.byref(rc), _p(rays[i], _F64P),
                         _p(out[i], _F64P))
    return out


def render(scene, camera, cfg, nthreads=0):
    """``render_view``'s per-pixel arrays for one camera: dict of rgb (H, W, 3),
    d_min, d_max, d_exp, z_surface (H, W) f32 and n_samples (H, W) i32."""
    st, _keep = _scene_struct(scene)
    rc = _cfg_struct(cfg)
    rot = _c(camera.rotation, np.float64)
    pos = _c(camera.position, np.float64)
    intr = np.array([camera.fx, camera.fy, camera.cx, camera.cy, camera.width, camera.height],
                    np.float64)
    h, w = int(camera.height), int(camera.width)
    o = dict(rgb=np.zeros((h, w, 3), np.float32), d_min=np.zeros((h, w), np.float32),
             d_max=np.zeros((h, w), np.float32), d_exp=np.zeros((h, w), np.float32),
             n_samples=np.zeros((h, w), np.int32), z_surface=np.zeros((h, w), np.float32))
    load().oracle_render(ctypes.byref(st), ctypes.byref(rc), _p(rot, _F64P), _p(pos, _F64P),
                         _p(intr, _F64P), _p(o["rgb"], _F32P), _p(o["d_min"], _F32P),
                         _p(o["d_max"], _F32P), _p(o["d_exp"], _F32P),
                         _p(o["n_samples"], _I32P), _p(o["z_surface"], _F32P),
                         nthreads or max_threads())
    return o


def bake(scene, g, half, origin, bounds=None, nthreads=0) -> np.ndarray:
    """``bake_density_grid`` values (G, G, G) f32; ``bounds`` = (min, max,
    unbounded) or a SceneBounds-like object."""
    st, _keep = _scene_struct(scene)
    origin = _c(origin, np.float64).reshape(3)
    dx = 2.0 * float(half) / int(g)                    # VoxelGrid.voxel_size
    unb = 0
    bc = np.zeros(3)
    bh = np.ones(3)
    if bounds is not None:
        lo, hi, unb = ((bounds.min, bounds.max, bounds.unbounded)
                       if hasattr(bounds, "unbounded") else bounds)
        lo, hi = np.asarray(lo, np.float64), np.asarray(hi, np.float64)
        bc, bh = 0.5 * (lo + hi), 0.5 * (hi - lo)      # SceneBounds.center / half
        unb = 1 if unb else 0
    out = np.zeros(int(g) ** 3, np.float32)
    load().oracle_bake(ctypes.byref(st), int(g), _p(origin, _F64P), dx, unb, _p(bc, _F64P),
                       _p(bh, _F64P), _p(out, _F32P), nthreads or max_threads())
    return out.reshape(int(g), int(g), int(g))
