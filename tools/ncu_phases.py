"""Per-function instruction / stall-sample totals of one kernel in an ncu report.

    python tools/ncu_phases.py <report.ncu-rep> [source.cu]

Reads the report's source page (cuda,sass view, -lineinfo builds) and charges
each CUDA source line of fuse.cu to the function that encloses it (inlined
helpers keep their own name), so the instruction mix of the pair kernel can
be compared across revisions.
"""
import csv
import io
import os
import re
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def func_ranges(lines):
    starts = []
    pat = re.compile(r"^(?:template <[^>]*>\s*)?(?:static |extern \"C\" )?(?:__device__|__global__|__host__)"
                     r"[^(]*?(\w+)\s*\(")
    for i, ln in enumerate(lines, 1):
        m = pat.match(ln)
        if m:
            starts.append((i, m.group(1)))
        elif ln.startswith("__global__") or ln.startswith("fuse_pairs("):
            pass
    # kernels written as "__global__ void __launch_bounds__(...)\nname(" : catch the name line
    for i, ln in enumerate(lines, 1):
        m = re.match(r"^(\w+)\((?:FuseConst|const)", ln)
        if m and i > 1 and "__global__" in lines[i - 2]:
            starts.append((i - 1, m.group(1)))
    starts.sort()
    return starts


def main():
    rep = sys.argv[1]
    src = sys.argv[2] if len(sys.argv) > 2 else os.path.join(ROOT, "paper_2601_04860_b200", "csrc",
                                                            "fuse.cu")
    out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source",
                          "cuda,sass"], capture_output=True, text=True).stdout
    base = os.path.basename(src)
    # the report's own copy of the source (--import-source), so line numbers
    # match the build that was profiled
    text = {}
    f = None
    full = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source",
                           "cuda"], capture_output=True, text=True).stdout
    for r in csv.reader(io.StringIO(full)):
        if r and r[0] in ("File Path", "File Name"):
            f = os.path.basename(r[1])
        elif f == base and len(r) > 1 and r[0].isdigit():
            text[int(r[0])] = r[1]
    lines = [text.get(i, "") for i in range(1, max(text) + 1)] if text else \
        open(src).read().splitlines()
    starts = func_ranges(lines)
    agg = {}
    f = None
    hdr = None
    for r in csv.reader(io.StringIO(out)):
        if not r:
            continue
        if r[0] == "File Path":
            f = os.path.basename(r[1])
            continue
        if r[0] == "Function Name":
            continue
        if r[0] == "Line No":
            hdr = r
            continue
        if hdr is None or len(r) < 9 or r[2] != "-":
            continue
        line = int(r[0])
        inst = int(r[7]) if r[7] not in ("-", "") else 0
        smp = int(r[4]) if r[4] not in ("-", "") else 0
        name = f
        if f == base:
            name = "?"
            for s, n in starts:
                if s <= line:
                    name = n
        a = agg.setdefault(name, [0, 0])
        a[0] += inst
        a[1] += smp
    ti = sum(v[0] for v in agg.values())
    ts = sum(v[1] for v in agg.values()) or 1
    print(f"total {ti / 1e6:.1f} M warp instructions")
    for k, v in sorted(agg.items(), key=lambda kv: -kv[1][0]):
        print(f"{k:28s} {v[0] / 1e6:7.1f}M {100 * v[0] / ti:5.1f}%   stall samples {100 * v[1] / ts:5.1f}%")


if __name__ == "__main__":
    main()
