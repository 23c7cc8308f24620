"""Build libdivas_b200.so (sm_100a) in-tree with nvcc.

    python -m paper_2601_04860_b200.build [--force] [--verbose]

Every translation unit is compiled with ``-fmad=false`` (no FMA contraction:
the reference's numba kernels emit none) and the IEEE
defaults for f64 division / sqrt (no fast-math).  The CUDA runtime is linked
statically, so the library needs only the driver at run time.
"""

from __future__ import annotations

import argparse
import concurrent.futures as cf
import os
import shutil
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
CSRC = os.path.join(HERE, "csrc")
LIBDIR = os.path.join(HERE, "_lib")
OBJDIR = os.path.join(LIBDIR, "obj")
LIB = os.path.join(LIBDIR, "libdivas_b200.so")
INCLUDE = os.path.join(os.path.dirname(HERE), "include")

SOURCES = ["abi.cu", "refine.cu", "fuse.cu", "threshold.cu", "overlay.cu", "render.cu"]
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
NVCC_FLAGS = ["-O3", "-lineinfo", "-std=c++17", "-fmad=false", "-prec-div=true",
              "-prec-sqrt=true", "-ftz=false", "-Xcompiler", "-fPIC,-O2",
              "-Xptxas", "-warn-spills", f"-I{INCLUDE}"]


def nvcc() -> str:
    for cand in (os.environ.get("NVCC"), "/usr/local/cuda/bin/nvcc", shutil.which("nvcc")):
        if cand and os.path.exists(cand):
            return cand
    raise RuntimeError("nvcc not found: the DivAS B200 kernels need the CUDA toolkit to build")


def _deps(src):
    headers = [os.path.join(CSRC, f) for f in os.listdir(CSRC) if f.endswith((".cuh", ".h"))]
    return [os.path.join(CSRC, src), os.path.join(INCLUDE, "divas_b200.h"), *headers]


def _stale(target, deps):
    if not os.path.exists(target):
        return True
    t = os.path.getmtime(target)
    return any(os.path.getmtime(d) > t for d in deps)


def _compile(src, verbose, objdir=None, defines=()):
    obj = os.path.join(objdir or OBJDIR, src.replace(".cu", ".o"))
    cmd = [nvcc(), *ARCH, *NVCC_FLAGS, *[f"-D{d}" for d in defines], "-c",
           os.path.join(CSRC, src), "-o", obj]
    if verbose:
        cmd.insert(1, "-Xptxas=-v")
    r = subprocess.run(cmd, capture_output=True, text=True)
    if r.returncode != 0:
        raise RuntimeError(f"nvcc failed on {src}:\n{r.stderr}")
    return obj, r.stderr


def build(force: bool = False, verbose: bool = False) -> str:
    os.makedirs(OBJDIR, exist_ok=True)
    todo = [s for s in SOURCES
            if force or _stale(os.path.join(OBJDIR, s.replace(".cu", ".o")), _deps(s))]
    logs = []
    if todo:
        with cf.ThreadPoolExecutor(max_workers=len(todo)) as ex:
            for obj, log in ex.map(lambda s: _compile(s, verbose), todo):
                logs.append(log)
    objs = [os.path.join(OBJDIR, s.replace(".cu", ".o")) for s in SOURCES]
    if force or todo or _stale(LIB, objs):
        tmp = LIB + ".tmp"
        cmd = [nvcc(), *ARCH, "-shared", "-o", tmp, *objs, "-cudart", "static"]
        r = subprocess.run(cmd, capture_output=True, text=True)
        if r.returncode != 0:
            raise RuntimeError(f"link failed:\n{r.stderr}")
        os.replace(tmp, LIB)
    if verbose:
        sys.stderr.write("".join(logs))
    return LIB


def build_variant(out_lib: str, defines) -> str:
    """Build an experiment variant (extra -D defines) to ``out_lib``; load it with
    DIVAS_LIB=<out_lib>.  Always a full rebuild into its own object dir."""
    objdir = out_lib + ".obj"
    os.makedirs(objdir, exist_ok=True)
    with cf.ThreadPoolExecutor(max_workers=len(SOURCES)) as ex:
        list(ex.map(lambda s: _compile(s, False, objdir, defines), SOURCES))
    objs = [os.path.join(objdir, s.replace(".cu", ".o")) for s in SOURCES]
    r = subprocess.run([nvcc(), *ARCH, "-shared", "-o", out_lib, *objs, "-cudart", "static"],
                       capture_output=True, text=True)
    if r.returncode != 0:
        raise RuntimeError(f"link failed:\n{r.stderr}")
    return out_lib


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--force", action="store_true")
    ap.add_argument("--verbose", action="store_true")
    ap.add_argument("--variant", help="output .so path for an experiment build")
    ap.add_argument("-D", dest="defines", action="append", default=[])
    args = ap.parse_args()
    if args.variant:
        print(build_variant(args.variant, args.defines))
    else:
        print(build(force=args.force, verbose=args.verbose))


if __name__ == "__main__":
    main()
