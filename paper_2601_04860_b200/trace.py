"""Per-pair public operations and the decision trace, on the device.

Mirrors of the reference's debugging surface
(/root/reference/pkg/src/divas/fusion.py):

* ``ThickPathDecision`` / ``ThinPathDecision`` (:126-162);
* ``thick_check`` (:549-603), ``thin_check`` (:606-646),
  ``depth_gradient`` (:516-520), ``depth_weight`` (:523-531);
* ``fuse_traced`` -- the ``fuse(trace_path=...)`` branch (:715-717,
  :727-764): one JSON line per (voxel, view) decision, probabilities from the
  traced decisions.

The pair evaluations run in ``divas_pair_trace`` (csrc/fuse.cu) with the
public functions' own arithmetic (f64 at the d_min/d_max sites because the
reference passes Python floats, true-size gradient neighbourhoods), which is
why -- exactly as in the reference -- the traced probabilities agree with
``fuse`` to ~1e-12 rather than bitwise (test_fusion.py:269-278).
``depth_weight`` is the reference's scalar formula (no array work).
"""

from __future__ import annotations

import ctypes
import json
import math
from dataclasses import asdict, dataclass

import numpy as np

from . import _native

__all__ = ["ThickPathDecision", "ThinPathDecision", "thick_check", "thin_check",
           "depth_gradient", "depth_weight", "fuse_traced"]

STAGES = ("frustum", "no-surface", "mask-gate", "density-gate", "spatial", "depth", "passed")

RECORD_DTYPE = np.dtype([
    ("stage", np.int32), ("thin_candidate", np.int32),
    ("m", np.float64), ("delta", np.float64), ("g", np.float64),
    ("tau_spatial", np.float64), ("tau_depth", np.float64), ("t_proj", np.float64),
    ("t_clamped", np.float64), ("x_d", np.float64), ("mu_d", np.float64), ("h_d", np.float64),
    ("r", np.float64), ("w_depth", np.float64),
    ("x_start", np.int64), ("x_end", np.int64), ("y_start", np.int64), ("y_end", np.int64),
    ("support_count", np.int64), ("n_pixels", np.int64),
    ("p_covered", np.float64), ("m_max", np.float64), ("t", np.float64),
])
assert RECORD_DTYPE.itemsize == 176


class _TraceArgs(ctypes.Structure):
    _VP = ctypes.c_void_p
    _fields_ = [
        ("nv", ctypes.c_int32), ("hm", ctypes.c_int32), ("wm", ctypes.c_int32),
        ("cams", _VP), ("masks", _VP), ("dmins", _VP), ("dmaxs", _VP), ("dexps", _VP),
        ("nsamps", _VP), ("pv", ctypes.c_double * 14), ("bc", ctypes.c_double * 3),
        ("bh", ctypes.c_double * 3), ("unbounded", ctypes.c_int32), ("dx_vox", ctypes.c_double),
        ("n", ctypes.c_int64), ("points", _VP), ("rho", _VP), ("views", _VP), ("out", _VP),
    ]


@dataclass
class ThickPathDecision:
    """Trace record for one (voxel, view) thick-path evaluation."""

    voxel: tuple
    view: int
    stage: str  # passed | frustum | no-surface | mask-gate | density-gate | spatial | depth
    m: float = 0.0
    delta: float = 0.0
    g: float = 0.0
    tau_spatial: float = 0.0
    tau_depth: float = 0.0
    t_proj: float = 0.0
    t_clamped: float = 0.0
    x_d: float = 0.0
    mu_d: float = 0.0
    h_d: float = 0.0
    r: float = 0.0
    w_depth: float = 0.0


@dataclass
class ThinPathDecision:
    """Trace record for one (voxel, view) thin-path evaluation."""

    voxel: tuple
    view: int
    candidate: bool
    x_start: int = 0
    x_end: int = -1
    y_start: int = 0
    y_end: int = -1
    support_count: int = 0
    n_pixels: int = 0
    p_covered: float = 0.0
    m_max: float = 0.0
    t: float = 0.0


def _records(dv, points, rho, views, params, bounds, voxel_size):
    """Run divas_pair_trace for query arrays; returns a numpy record array."""
    import torch
    from .fusion import _params_vector, bounds_arrays
    dev = dv.device
    n = len(rho)
    out = torch.empty(n * RECORD_DTYPE.itemsize, dtype=torch.uint8, device=dev)
    pts = torch.from_numpy(np.ascontiguousarray(points, np.float64)).to(dev)
    rh = torch.from_numpy(np.ascontiguousarray(rho, np.float64)).to(dev)
    vw = torch.from_numpy(np.ascontiguousarray(views, np.int32)).to(dev)
    bc, bh, unb = bounds_arrays(bounds)
    a = _TraceArgs()
    a.nv, a.hm, a.wm = dv.nv, dv.hm, dv.wm
    a.cams = _native.ptr(dv.cams)
    a.masks, a.dmins, a.dmaxs = _native.ptr(dv.masks), _native.ptr(dv.dmins), _native.ptr(dv.dmaxs)
    a.dexps, a.nsamps = _native.ptr(dv.dexps), _native.ptr(dv.nsamps)
    a.pv[:] = _params_vector(params).tolist()
    a.bc[:], a.bh[:] = list(bc), list(bh)
    a.unbounded = int(unb)
    a.dx_vox = float(voxel_size)
    a.n = n
    a.points, a.rho, a.views, a.out = (_native.ptr(t) for t in (pts, rh, vw, out))
    lib = _native.lib()
    _native.check(lib.divas_pair_trace(ctypes.byref(a), _native.stream_handle()),
                  "divas_pair_trace")
    return out.cpu().numpy().view(RECORD_DTYPE)


def _single_view(view, mask):
    from .fusion import DeviceViews
    return DeviceViews.from_views([(view, mask)])


def _thick_dec(rec, voxel_index, view_index):
    stage = STAGES[int(rec["stage"])]
    dec = ThickPathDecision(voxel=tuple(voxel_index), view=view_index, stage=stage)
    if stage in ("frustum", "no-surface"):
        return dec
    dec.m = float(rec["m"])
    dec.x_d = float(rec["x_d"])
    if stage in ("mask-gate", "density-gate"):
        return dec
    for f in ("delta", "g", "tau_spatial", "tau_depth", "t_proj", "t_clamped", "mu_d", "h_d",
              "r", "w_depth"):
        setattr(dec, f, float(rec[f]))
    return dec


def _thin_dec(rec, voxel_index, view_index):
    dec = ThinPathDecision(voxel=tuple(voxel_index), view=view_index, candidate=False)
    if not rec["thin_candidate"]:
        return dec
    dec.candidate = True
    dec.x_start, dec.x_end = int(rec["x_start"]), int(rec["x_end"])
    dec.y_start, dec.y_end = int(rec["y_start"]), int(rec["y_end"])
    dec.support_count, dec.n_pixels = int(rec["support_count"]), int(rec["n_pixels"])
    dec.p_covered, dec.m_max, dec.t = float(rec["p_covered"]), float(rec["m_max"]), float(rec["t"])
    return dec


def thick_check(voxel_center, voxel_size, rho, view, mask, params, bounds=None,
                voxel_index=(0, 0, 0), view_index=0):
    """fusion.py:549-603: (passed, ThickPathDecision) for one voxel and view."""
    rec = _records(_single_view(view, mask), np.asarray(voxel_center, np.float64).reshape(1, 3),
                   [float(rho)], [0], params, bounds, voxel_size)[0]
    dec = _thick_dec(rec, voxel_index, view_index)
    return dec.stage == "passed", dec


def thin_check(voxel_center, voxel_size, rho, view, mask, params, voxel_index=(0, 0, 0),
               view_index=0):
    """fusion.py:606-646: ThinPathDecision for one voxel and view."""
    rec = _records(_single_view(view, mask), np.asarray(voxel_center, np.float64).reshape(1, 3),
                   [float(rho)], [0], params, None, voxel_size)[0]
    return _thin_dec(rec, voxel_index, view_index)


def depth_gradient(view, pixel, eps: float = 1e-8, kappa: float = 1.0) -> float:
    """fusion.py:516-520: the depth-gradient factor at a pixel of ``view``."""
    import torch
    from ._device import as_device, device
    dev = device()
    h, w = np.asarray(view.d_exp).shape
    planes = [as_device(np.asarray(a)[None], dt, dev) for a, dt in
              ((view.d_exp, np.float32), (view.d_min, np.float32), (view.d_max, np.float32),
               (view.n_samples, np.int32))]
    out = torch.empty((1, h, w), dtype=torch.float64, device=dev)
    lib = _native.lib()
    _native.check(lib.divas_gradient_maps(1, h, w, *(_native.ptr(p) for p in planes), float(eps),
                                          float(kappa), 0, _native.ptr(out),
                                          _native.stream_handle()), "divas_gradient_maps")
    ix, iy = int(pixel[0]), int(pixel[1])
    return float(out[0, iy, ix].item())


def depth_weight(t_clamped: float, d_min: float, d_max: float, alpha1: float,
                 eps: float = 1e-8) -> float:
    """fusion.py:523-531 (scalar formula)."""
    if d_min > d_max:
        raise ValueError("d_min must not exceed d_max")
    mu = 0.5 * (d_min + d_max)
    hd = max(0.5 * (d_max - d_min), eps)
    r = abs(t_clamped - mu) / hd
    return math.exp(-alpha1 * r * r)


def fuse_traced(grid, density, views, params, bounds, trace_path, chunk_voxels=1 << 16):
    """fusion.py:727-764 on the device: one JSON line per decision, in the
    reference's (voxel C-order, view) order; returns the traced probabilities."""
    from .fusion import DeviceViews
    g = int(grid.resolution)
    dx = float(grid.voxel_size())
    origin = np.asarray(grid.origin, dtype=np.float64).reshape(3)
    dens = np.asarray(density.values, dtype=np.float32).reshape(-1)
    pv = np.asarray(params.as_vector(), dtype=np.float64)
    eps, thin_accept, enable_thin = pv[9], pv[8], pv[13] != 0.0
    nv = len(views)
    dv = DeviceViews.from_views(views)
    probs = np.zeros(g ** 3)
    with open(trace_path, "w") as fout:
        for lo in range(0, g ** 3, chunk_voxels):
            hi = min(lo + chunk_voxels, g ** 3)
            vi = np.arange(lo, hi)
            ix, rem = np.divmod(vi, g * g)
            iy, iz = np.divmod(rem, g)
            idx = np.stack([ix, iy, iz], axis=1)
            centers = origin + (idx.astype(np.float64) + 0.5) * dx     # VoxelGrid.index_to_center
            pts = np.repeat(centers, nv, axis=0)
            rho = np.repeat(dens[lo:hi].astype(np.float64), nv)
            vws = np.tile(np.arange(nv, dtype=np.int32), hi - lo)
            recs = _records(dv, pts, rho, vws, params, bounds, dx).reshape(hi - lo, nv)
            for k in range(hi - lo):
                vox = (int(idx[k, 0]), int(idx[k, 1]), int(idx[k, 2]))
                tw, tmw, tt = [], [], []
                for view_i in range(nv):
                    rec = recs[k, view_i]
                    dec = _thick_dec(rec, vox, view_i)
                    if dec.stage not in ("frustum", "no-surface"):
                        fout.write(json.dumps({"path": "thick", **asdict(dec)}) + "\n")
                    if dec.stage == "passed":
                        tw.append(dec.w_depth)
                        tmw.append(dec.m * dec.w_depth)
                        continue
                    if dec.stage in ("frustum", "no-surface") or not enable_thin:
                        continue
                    tdec = _thin_dec(rec, vox, view_i)
                    if tdec.candidate:
                        fout.write(json.dumps({"path": "thin", **asdict(tdec)}) + "\n")
                        if tdec.n_pixels > 0 and tdec.t >= thin_accept:
                            tt.append(tdec.t)
                order = sorted(range(len(tw)), key=lambda j: (tw[j], tmw[j]))
                sw = sum(tw[j] for j in order)
                smw = sum(tmw[j] for j in order)
                st = sum(sorted(tt))
                denom = sw + len(tt)
                probs[lo + k] = (smw + st) / denom if denom > eps else 0.0
    return probs.reshape(g, g, g)
