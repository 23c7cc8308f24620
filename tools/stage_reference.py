"""Stage the unmodified reference for the bench's reference arm and the
drop-in acceptance suite (run in a container that has /root/reference).

    python tools/stage_reference.py

* ``baseline/_ref/``: ``pip install --no-index --no-build-isolation --no-deps``
  of a copy of /root/reference/pkg (its build writes into the source tree,
  and /root/reference is read-only), i.e. the ``divas`` package itself;
* ``baseline/_ref/_tests/``: the reference's own test files, which
  ``tests/test_reference_suite.py`` runs with the B200 swap installed.

``baseline/`` is git-ignored (not product source) but is not gpurun-ignored,
so it travels to the GPU box with the snapshot; nothing is copied into the
repo's tracked tree.
"""
import os
import shutil
import subprocess
import sys
import tempfile

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
SRC = "/root/reference/pkg"
DST = os.path.join(ROOT, "baseline", "_ref")


def main():
    if not os.path.isdir(SRC):
        sys.exit(f"{SRC} not found: stage the reference in the build container")
    tmp = tempfile.mkdtemp()
    pkg = os.path.join(tmp, "pkg")
    shutil.copytree(SRC, pkg)
    shutil.rmtree(DST, ignore_errors=True)
    subprocess.run([sys.executable, "-m", "pip", "install", "--no-index", "--no-build-isolation",
                    "--no-deps", "--find-links", "/opt/wheelhouse", "--target", DST, pkg],
                   check=True)
    shutil.copytree(os.path.join(SRC, "tests"), os.path.join(DST, "_tests"))
    shutil.rmtree(tmp, ignore_errors=True)
    print(f"staged divas into {DST} (+ _tests)")


if __name__ == "__main__":
    main()
