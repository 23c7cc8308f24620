"""The reference's own tests, run with the B200 path swapped in (drop-in acceptance).

SURVEY.md section 4 / 8b ("Swap mechanics") name these as the drop-in gate:
``test_fusion.py`` (/root/reference/pkg/tests/test_fusion.py:201-316 and the
rest of the file), ``test_segmenter.py::TestRefineMask`` (:93-141), acceptance
criterion #1 (``test_acceptance.py:130-145``: ``fuse`` vs ``fuse_reference``
< 1e-6 over 200 random instances) and #8 (``:290-302``: byte-identical
``.vgrid`` across worker counts).

Each level of INTEGRATION.md is installed exactly as documented, through
``paper_2601_04860_b200.integration``:

* level A: ``divas.fusion._fuse_kernel`` -> ``fuse_kernel_b200`` (ctypes over
  the C ABI), so every ``fuse`` call runs the device kernel;
* level B: the by-name rebinding of ``fuse`` / ``refine_mask`` /
  ``project_grid_overlay`` in the reference's modules and in each test module
  (they did ``from divas.fusion import fuse``).

The reference package comes from ``baseline/_ref`` (``tools/stage_reference.py``:
pip-installed /root/reference/pkg plus a copy of its tests, git-ignored, shipped
to the GPU box with the snapshot); without it the test skips and says why.
"""

import os
import re
import shutil
import subprocess
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
REF = os.path.join(ROOT, "baseline", "_ref")
REF_TESTS = os.path.join(REF, "_tests")

SELECTION = [
    "test_fusion.py",
    "test_segmenter.py::TestRefineMask",
    "test_acceptance.py::test_criterion_1_oracle_equivalence",
    "test_acceptance.py::test_criterion_8_determinism",
]
# none of the selected tests is a known reference failure (SURVEY.md section 4:
# the two known unit failures are in test_session.py / test_cli.py, and #9 is
# not selected), so every selected test must pass with the swap installed
ALLOWED_FAILURES = set()

CONFTEST = '''
import os
import sys

sys.path.insert(0, {ref!r})
sys.path.insert(1, {root!r})

import divas  # noqa: E402
from paper_2601_04860_b200 import integration  # noqa: E402

LEVEL = os.environ["DIVAS_SWAP"]
if LEVEL == "A":
    integration.install_operator_swap(divas)
else:
    integration.install_api_swap(divas)


def pytest_collection_modifyitems(session, config, items):
    if LEVEL != "B":
        return
    seen = set()
    for it in items:
        mod = getattr(it, "module", None)
        if mod is not None and id(mod) not in seen:
            seen.add(id(mod))
            integration.patch_namespace(mod.__dict__)


def pytest_sessionfinish(session, exitstatus):
    import divas.fusion
    # prove which implementation ran
    fk = divas.fusion._fuse_kernel.__name__
    fz = getattr(divas.fusion.fuse, "__module__", "?")
    print(f"\\nSWAP-CHECK level={{LEVEL}} _fuse_kernel={{fk}} fuse_module={{fz}}")
'''


def _have_reference():
    return os.path.isdir(os.path.join(REF, "divas")) and os.path.isdir(REF_TESTS)


@pytest.mark.gpu
@pytest.mark.parametrize("level", ["A", "B"])
def test_reference_suite_with_swap(level, tmp_path):
    if not _have_reference():
        pytest.skip("baseline/_ref (the pip-installed reference + its tests) is not staged: "
                    "run tools/stage_reference.py where /root/reference exists")
    import torch
    assert torch.cuda.is_available(), "the swap runs the device kernels"
    tdir = tmp_path / "tests"
    shutil.copytree(REF_TESTS, tdir)
    (tdir / "conftest.py").write_text(CONFTEST.format(ref=REF, root=ROOT))
    env = dict(os.environ)
    env["DIVAS_SWAP"] = level
    env["PYTHONPATH"] = os.pathsep.join([REF, ROOT])
    env.setdefault("NUMBA_CACHE_DIR", "/tmp/divas_ref_numba_cache")
    cmd = [sys.executable, "-m", "pytest", "-q", "-rf", "-s", "-p", "no:cacheprovider",
           "--import-mode=importlib", *[str(tdir / s) for s in SELECTION]]
    r = subprocess.run(cmd, cwd=str(tmp_path), env=env, capture_output=True, text=True,
                       timeout=1800)
    out = r.stdout + r.stderr
    tail = "\n".join(out.splitlines()[-40:])
    failed = set(re.findall(r"^FAILED (\S+)", out, re.M))
    failed = {f.split("tests/", 1)[-1] for f in failed}
    assert f"SWAP-CHECK level={level}" in out, tail
    if level == "A":
        assert "_fuse_kernel=fuse_kernel_b200" in out, tail
    else:
        assert "fuse_module=paper_2601_04860_b200.fusion" in out, tail
    m = re.search(r"(\d+) passed", out)
    assert m and int(m.group(1)) > 30, tail
    assert failed <= ALLOWED_FAILURES, f"unexpected failures {sorted(failed)}\n{tail}"
    assert r.returncode in (0, 1), tail
    print(f"level {level}: {m.group(0)}, failures {sorted(failed) or 'none'}")
