"""ctypes binding of libdivas_b200.so (the C ABI declared in include/divas_b200.h).

There is no CPU fallback: if the library is missing or no CUDA device is
present, every compute entry point raises.  Build it with
``python -m paper_2601_04860_b200.build`` (``__graft_entry__.build()`` does).
"""

from __future__ import annotations

import ctypes
import os
import threading

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("DIVAS_LIB") or os.path.join(_HERE, "_lib", "libdivas_b200.so")

CAM_STRIDE = 18
NPARAM = 14

# every symbol include/divas_b200.h declares
EXPORTS = (
    "divas_refine_workspace_size", "divas_refine", "divas_records_size", "divas_bands_size",
    "divas_refine_bands",
    "divas_fuse_workspace_size", "divas_fuse_workspace_size_ext", "divas_fuse", "divas_gate_count",
    "divas_fuse_gated_count",
    "divas_fuse_overflow", "divas_fuse_ws_regions",
    "divas_gradient_maps", "divas_pair_trace",
    "divas_threshold_workspace_size", "divas_threshold",
    "divas_overlay", "divas_vgrid_payload",
    "divas_last_error", "divas_abi_version", "divas_refine_bands_roi", "divas_refine_minmax",
    "divas_refine_bands_keys", "divas_copy2d_h2d", "divas_gather2d_h2d", "divas_peer_put",
    "divas_render", "divas_march_rays", "divas_bake_density", "divas_mask_bbox",
)

_VP = ctypes.c_void_p
_D3 = ctypes.c_double * 3


class FuseArgs(ctypes.Structure):
    """Mirror of ``divas_fuse_args`` (include/divas_b200.h)."""

    _fields_ = [
        ("g", ctypes.c_int64), ("origin", _D3), ("dx_vox", ctypes.c_double),
        ("density", _VP), ("nv", ctypes.c_int32), ("hm", ctypes.c_int32),
        ("wm", ctypes.c_int32), ("cams", _VP), ("masks", _VP), ("dmins", _VP),
        ("dmaxs", _VP), ("dexps", _VP), ("nsamps", _VP),
        ("pv", ctypes.c_double * NPARAM), ("bc", _D3), ("bh", _D3),
        ("unbounded", ctypes.c_int32), ("vox_lo", ctypes.c_int64), ("vox_hi", ctypes.c_int64),
        ("probs", _VP), ("n_thick", _VP), ("n_thin", _VP), ("sw", _VP), ("smw", _VP),
        ("st", _VP), ("occ", _VP), ("occ_thr", ctypes.c_double), ("max_gated", ctypes.c_int64),
        ("records", _VP), ("bands", _VP), ("nv_cap", ctypes.c_int32), ("mode", ctypes.c_int32),
        ("view_lo", ctypes.c_int32), ("view_hi", ctypes.c_int32),
        ("occ_peers", _VP), ("n_peers", ctypes.c_int32), ("fallbacks", _VP),
    ]

MAX_PRIMS = 128


class Copy2D(ctypes.Structure):
    """Mirror of ``divas_copy2d`` (one rectangle of divas_gather2d_h2d)."""

    _fields_ = [("src", _VP), ("dst", _VP), ("spitch", ctypes.c_int64),
                ("dpitch", ctypes.c_int64), ("width_bytes", ctypes.c_int64),
                ("rows", ctypes.c_int64)]


class Scene(ctypes.Structure):
    """Mirror of ``divas_scene`` (host arrays; the struct is copied into the launch)."""

    _fields_ = [("n_prims", ctypes.c_int32), ("kinds", _VP), ("params", _VP),
                ("density", _VP), ("colors", _VP), ("soft", _VP), ("background", _D3)]


class RenderCfg(ctypes.Structure):
    """Mirror of ``divas_render_cfg``."""

    _fields_ = [("samples_per_ray", ctypes.c_int32), ("near_", ctypes.c_double),
                ("far_", ctypes.c_double), ("tau_cw", ctypes.c_double),
                ("min_weight", ctypes.c_double)]


# fallback counters (divas_fuse_args.fallbacks), DIVAS_FB_* in the header
FALLBACKS = ("centre", "thick", "thick_t", "corners", "recount", "thin_gate", "band_wide",
             "tile_skip", "thin_sort")
NFALLBACK = 9

FUSE_FULL = 0
STEP_GATE, STEP_CLEAR_ALL, STEP_CLEAR_VIEWS, STEP_PAIRS, STEP_REDUCE = 1, 2, 4, 8, 16
STEP_ZERO, STEP_GATE_KEEP = 32, 64
FUSE_INCREMENTAL = STEP_CLEAR_VIEWS | STEP_PAIRS | STEP_REDUCE


_lib = None
_lock = threading.Lock()


def _declare(lib):
    S, I64, I32, D = ctypes.c_size_t, ctypes.c_int64, ctypes.c_int32, ctypes.c_double
    sig = {
        "divas_refine_workspace_size": (S, [I32]),
        "divas_refine": (ctypes.c_int, [I32, I64, I64, _VP, _VP, _VP, _VP, _VP, S, _VP]),
        "divas_records_size": (S, [I32, I64, I64]),
        "divas_bands_size": (S, [I32, I64, I64]),
        "divas_refine_bands": (ctypes.c_int, [I32, I64, I64, _VP, _VP, _VP, _VP, _VP,
                                              ctypes.POINTER(D), D, _VP, _VP, _VP, S, _VP]),
        "divas_refine_bands_roi": (ctypes.c_int, [I32, I64, I64, _VP, _VP, _VP, _VP, _VP,
                                                  ctypes.POINTER(D), D, _VP, _VP, _VP, S, _VP,
                                                  I32, I32, _VP]),
        "divas_refine_minmax": (ctypes.c_int, [I32, I64, I64, _VP, _VP, _VP, _VP]),
        "divas_copy2d_h2d": (ctypes.c_int, [_VP, S, _VP, S, S, S, _VP]),
        "divas_gather2d_h2d": (ctypes.c_int, [ctypes.POINTER(Copy2D), I32, _VP]),
        "divas_mask_bbox": (ctypes.c_int, [I32, I64, I64, _VP, ctypes.c_float, _VP, _VP]),
        "divas_peer_put": (ctypes.c_int, [_VP, S, _VP, I32, S, _VP]),
        "divas_refine_bands_keys": (ctypes.c_int, [I32, I64, I64, _VP, _VP, _VP, _VP, _VP,
                                                   ctypes.POINTER(D), D, _VP, _VP, _VP, _VP, S,
                                                   _VP, I32, I32, _VP]),
        "divas_fuse_workspace_size": (S, [I64, I32, I32, I32]),
        "divas_fuse_workspace_size_ext": (S, [I64, I32, I32, I32, I32]),
        "divas_fuse": (ctypes.c_int, [ctypes.POINTER(FuseArgs), _VP, S, _VP]),
        "divas_gate_count": (ctypes.c_int, [ctypes.POINTER(FuseArgs), _VP, _VP]),
        "divas_fuse_gated_count": (_VP, [_VP]),
        "divas_fuse_overflow": (_VP, [_VP]),
        "divas_fuse_ws_regions": (None, [I64, I32, I32, I32, I32, ctypes.POINTER(S)]),
        "divas_gradient_maps": (ctypes.c_int, [I32, I32, I32, _VP, _VP, _VP, _VP, D, D, I32, _VP,
                                               _VP]),
        "divas_pair_trace": (ctypes.c_int, [_VP, _VP]),
        "divas_threshold_workspace_size": (S, [I64]),
        "divas_threshold": (ctypes.c_int, [_VP, I64, D, I64, _VP, _VP, _VP, _VP, S, _VP]),
        "divas_overlay": (ctypes.c_int, [_VP, I32, I32, _VP, _VP, _VP, _VP, I64,
                                         ctypes.POINTER(D), D, ctypes.POINTER(D),
                                         ctypes.POINTER(D), I32, D, _VP, _VP]),
        "divas_vgrid_payload": (ctypes.c_int, [_VP, I64, _VP, _VP]),
        "divas_render": (ctypes.c_int, [ctypes.POINTER(Scene), ctypes.POINTER(RenderCfg), I32,
                                        _VP, I32, I32, _VP, _VP, _VP, _VP, _VP, _VP, _VP, _VP]),
        "divas_march_rays": (ctypes.c_int, [ctypes.POINTER(Scene), ctypes.POINTER(RenderCfg),
                                            I64, _VP, _VP, _VP, _VP, _VP]),
        "divas_bake_density": (ctypes.c_int, [ctypes.POINTER(Scene), I64, ctypes.POINTER(D), D,
                                              I32, ctypes.POINTER(D), ctypes.POINTER(D), _VP,
                                              _VP]),
        "divas_last_error": (ctypes.c_char_p, []),
        "divas_abi_version": (ctypes.c_int, []),
    }
    for name, (res, args) in sig.items():
        fn = getattr(lib, name, None)
        if fn is None and os.environ.get("DIVAS_LIB"):
            continue      # experiment builds of older revisions (tools/ab.sh)
        if fn is None:
            raise RuntimeError(f"{LIB_PATH} does not export {name}: rebuild the library")
        fn.restype = res
        fn.argtypes = args


def lib():
    """The loaded library; raises if it has not been built (no fallback)."""
    global _lib
    with _lock:
        if _lib is None:
            if not os.path.exists(LIB_PATH):
                raise RuntimeError(
                    f"{LIB_PATH} is missing: build the sm_100a kernels with "
                    "`python -m paper_2601_04860_b200.build` (there is no CPU fallback)")
            handle = ctypes.CDLL(LIB_PATH)
            _declare(handle)
            _lib = handle
    return _lib


def ws_regions(cap, nv_cap, hm, wm, internal_aux=False):
    """Byte offsets {work, bits_thick, bits_thin, w, mw, t, total} of a fuse
    workspace (``internal_aux``: room for records / bands built by divas_fuse)."""
    out = (ctypes.c_size_t * 7)()
    lib().divas_fuse_ws_regions(int(cap), int(nv_cap), int(hm), int(wm), int(bool(internal_aux)),
                                out)
    return dict(zip(("work", "bits_thick", "bits_thin", "w", "mw", "t", "total"), list(out)))


def check(rc: int, what: str):
    if rc != 0:
        msg = lib().divas_last_error().decode(errors="replace")
        if rc == 1:
            raise ValueError(f"{what}: {msg}")
        raise RuntimeError(f"{what} failed (code {rc}): {msg}")


def ptr(t) -> int:
    """Device pointer of a torch tensor (0 for None)."""
    return 0 if t is None else int(t.data_ptr())


def stream_handle(stream=None) -> int:
    import torch
    s = stream if stream is not None else torch.cuda.current_stream()
    return int(s.cuda_stream)
