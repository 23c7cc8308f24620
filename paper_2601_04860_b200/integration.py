"""Drop-in installers for the reference package (``divas``): INTEGRATION.md A and B.

``install_operator_swap(divas)`` (level A) replaces ``divas.fusion._fuse_kernel``
-- the numba operator that ``divas.fusion.fuse`` resolves as a module global
at call time (/root/reference/pkg/src/divas/fusion.py:708-723) -- with
``fuse_kernel_b200``, a ctypes call of ``divas_fuse`` over the C ABI
(include/divas_b200.h) with the same signature and output contract
(fusion.py:494-496).  Every caller of ``fuse`` (session, ablation, CLI, the
reference's tests) then runs the B200 kernel.

``install_api_swap(divas)`` (level B) rebinds the reference's public names
(``fuse``, ``refine_mask``, ``project_grid_overlay``) in every module that
bound them, to this package's mirrors, which take the reference's own
objects.  ``patch_namespace(ns)`` applies the same rebinding to any other
namespace that did ``from divas.fusion import fuse`` (a test module, say).

Both are exercised by ``tests/test_reference_suite.py``, which runs the
reference's own tests with each swap installed.
"""

from __future__ import annotations

import ctypes

import numpy as np

from . import _native

__all__ = ["fuse_kernel_b200", "install_operator_swap", "install_api_swap", "patch_namespace",
           "API_NAMES"]


def fuse_kernel_b200(g, origin, dx_vox, density, rots, poss, intr, masks, dmins, dmaxs, dexps,
                     nsamps, valids, gmaps, pv, bc, bh, unbounded, n_chunks, out):
    """``divas.fusion._fuse_kernel`` on the device (fusion.py:493-509): fills
    ``out[G^3]`` with p.  ``gmaps``, ``valids`` and ``n_chunks`` are not read:
    the kernel derives the gradient and valid = n > 0 itself, and its result
    does not depend on a worker split (as the reference's does not)."""
    import torch
    if not torch.cuda.is_available():
        raise RuntimeError("fuse_kernel_b200 needs a CUDA device (there is no CPU path)")
    dev = torch.device("cuda", torch.cuda.current_device())
    g = int(g)
    nv, hm, wm = (int(x) for x in masks.shape)

    def t(a, dt=None):
        return torch.from_numpy(np.ascontiguousarray(a, dtype=dt)).to(dev)

    cams = t(np.concatenate([np.asarray(rots, np.float64).reshape(nv, 9),
                             np.asarray(poss, np.float64).reshape(nv, 3),
                             np.asarray(intr, np.float64).reshape(nv, 6)], axis=1))
    planes = [t(masks, np.float32), t(dmins, np.float32), t(dmaxs, np.float32),
              t(dexps, np.float32), t(nsamps, np.int32)]
    dens = t(np.asarray(density).reshape(-1), np.float32)
    probs = torch.empty(g ** 3, dtype=torch.float64, device=dev)
    lib = _native.lib()
    a = _native.FuseArgs()
    a.g, a.dx_vox, a.nv, a.hm, a.wm = g, float(dx_vox), nv, hm, wm
    a.origin[:] = [float(x) for x in np.asarray(origin).reshape(3)]
    a.pv[:] = [float(x) for x in np.asarray(pv).reshape(-1)[:_native.NPARAM]]
    a.bc[:] = [float(x) for x in np.asarray(bc).reshape(3)]
    a.bh[:] = [float(x) for x in np.asarray(bh).reshape(3)]
    a.unbounded, a.vox_lo, a.vox_hi = int(unbounded), 0, g ** 3
    a.density, a.cams, a.probs = dens.data_ptr(), cams.data_ptr(), probs.data_ptr()
    a.masks, a.dmins, a.dmaxs, a.dexps, a.nsamps = (p.data_ptr() for p in planes)
    a.occ_thr = 0.5
    stream = torch.cuda.current_stream().cuda_stream
    hdr = torch.zeros(256, dtype=torch.uint8, device=dev)   # exact gated count sizes the workspace
    _native.check(lib.divas_gate_count(ctypes.byref(a), ctypes.c_void_p(hdr.data_ptr()),
                                       ctypes.c_void_p(stream)), "divas_gate_count")
    a.max_gated = max(int(hdr[:8].view(torch.int64).item()), 1)
    ws_bytes = int(lib.divas_fuse_workspace_size(a.max_gated, nv, hm, wm))
    ws = torch.empty(ws_bytes, dtype=torch.uint8, device=dev)
    _native.check(lib.divas_fuse(ctypes.byref(a), ctypes.c_void_p(ws.data_ptr()),
                                 ctypes.c_size_t(ws_bytes), ctypes.c_void_p(stream)), "divas_fuse")
    out[:] = probs.cpu().numpy()


# public names a by-name swap rebinds, and the package attribute that serves each
API_NAMES = {"fuse": "fuse", "refine_mask": "refine_mask",
             "project_grid_overlay": "project_grid_overlay"}


def install_operator_swap(divas) -> None:
    """Level A: ``divas.fusion._fuse_kernel = fuse_kernel_b200``."""
    import divas.fusion  # noqa: F401  (the submodule must be loaded)
    divas.fusion._fuse_kernel = fuse_kernel_b200


def patch_namespace(ns: dict) -> list:
    """Rebind the API_NAMES found in ``ns`` (a module's globals) to this
    package's mirrors; returns the names rebound."""
    import paper_2601_04860_b200 as b200
    done = []
    for name, attr in API_NAMES.items():
        if name in ns and callable(ns[name]) and getattr(ns[name], "__module__", "").startswith(
                "divas"):
            ns[name] = getattr(b200, attr)
            done.append(name)
    return done


def install_api_swap(divas) -> None:
    """Level B: rebind ``fuse`` / ``refine_mask`` / ``project_grid_overlay`` in
    every reference module that bound them ("Swap
    mechanics": fusion, segmenter, session, ablation, cli)."""
    import importlib
    for sub in ("fusion", "segmenter", "session", "ablation", "cli", "scenes"):
        try:
            mod = importlib.import_module(f"divas.{sub}")
        except ImportError:
            continue
        patch_namespace(mod.__dict__)
