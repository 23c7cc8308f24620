"""Host-side checks of the drop-in installers:
the reference package (baseline/_ref, when staged) gets its names rebound to
this package's mirrors, and nothing falls back to a CPU path."""

import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
REF = os.path.join(ROOT, "baseline", "_ref")

pytestmark = pytest.mark.skipif(not os.path.isdir(os.path.join(REF, "divas")),
                                reason="baseline/_ref not staged (tools/stage_reference.py)")


def _fresh_divas():
    for k in [k for k in sys.modules if k == "divas" or k.startswith("divas.")]:
        del sys.modules[k]
    if REF not in sys.path:
        sys.path.insert(0, REF)
    os.environ.setdefault("NUMBA_CACHE_DIR", "/tmp/divas_ref_numba_cache")
    import divas
    return divas


def test_operator_swap_rebinds_fuse_kernel():
    divas = _fresh_divas()
    import divas.fusion
    from paper_2601_04860_b200 import integration
    orig = divas.fusion._fuse_kernel
    integration.install_operator_swap(divas)
    try:
        assert divas.fusion._fuse_kernel is integration.fuse_kernel_b200
    finally:
        divas.fusion._fuse_kernel = orig


def test_api_swap_rebinds_public_names():
    divas = _fresh_divas()
    import importlib

    import paper_2601_04860_b200 as b200
    from paper_2601_04860_b200 import integration
    integration.install_api_swap(divas)
    fusion = importlib.import_module("divas.fusion")
    segmenter = importlib.import_module("divas.segmenter")
    session = importlib.import_module("divas.session")
    assert fusion.fuse is b200.fuse
    assert fusion.project_grid_overlay is b200.project_grid_overlay
    assert segmenter.refine_mask is b200.refine_mask
    assert session.fuse is b200.fuse and session.refine_mask is b200.refine_mask
    # fuse_reference stays the reference's CPU oracle
    ref = importlib.import_module("divas.reference")
    assert ref.fuse_reference.__module__ == "divas.reference"
    _fresh_divas()                         # leave an unpatched package behind


def test_patch_namespace_only_touches_reference_bindings():
    from paper_2601_04860_b200 import integration

    def fuse():                            # a local function named fuse: not the reference's
        return None
    ns = {"fuse": fuse, "other": 1}
    assert integration.patch_namespace(ns) == []
    assert ns["fuse"] is fuse
    divas = _fresh_divas()
    import divas.fusion
    ns = {"fuse": divas.fusion.fuse, "refine_mask": divas.segmenter.refine_mask}
    done = integration.patch_namespace(ns)
    import paper_2601_04860_b200 as b200
    assert sorted(done) == ["fuse", "refine_mask"]
    assert ns["fuse"] is b200.fuse and ns["refine_mask"] is b200.refine_mask


def test_operator_kernel_has_no_cpu_path():
    import numpy as np
    import torch
    from paper_2601_04860_b200 import integration
    if torch.cuda.is_available():
        pytest.skip("CPU-only check")
    with pytest.raises(RuntimeError):
        integration.fuse_kernel_b200(1, np.zeros(3), 1.0, np.zeros(1, np.float32),
                                     np.eye(3)[None], np.zeros((1, 3)), np.ones((1, 6)),
                                     np.zeros((1, 1, 1), np.float32), *([None] * 11),
                                     np.zeros(1))
