"""Per-function instruction attribution of an ncu --set full report (source page).

    python tools/ncu_funcs.py <ncu-rep> <kernel-substring> [--lib path.so] [--top N]

Maps each SASS address to its CUDA source line (nvdisasm line info of the
library the report was taken with) and the line to the enclosing function of
the .cu/.cuh file; prints warp instructions, thread instructions, lane
efficiency (thread / (32 warp)) and stall samples per function.
"""
import argparse
import csv
import io
import os
import re
import subprocess
import sys
from collections import defaultdict

sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))
import sass_lines  # noqa: E402

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
FUNC_RE = re.compile(r'^(?:template\s*<[^>]*>\s*)?(?:static\s+)?(?:__device__|__global__|__host__)'
                     r'[^(]*?\b(\w+)\s*\(')


def func_table(path):
    out = []
    for i, line in enumerate(open(path), 1):
        m = FUNC_RE.match(line)
        if m:
            out.append((i, m.group(1)))
    return out


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("rep")
    ap.add_argument("kernel")
    ap.add_argument("--lib", default=None)
    ap.add_argument("--top", type=int, default=30)
    a = ap.parse_args()
    if a.lib:
        sass_lines.LIB = a.lib
    lm = sass_lines.line_map(a.kernel)
    src = subprocess.run(["ncu", "-i", a.rep, "--page", "source", "--csv", "--print-source", "sass"],
                         capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(src)))
    hdr = rows[1]
    ia, iex = hdr.index("Address"), hdr.index("Instructions Executed")
    ith = hdr.index("Thread Instructions Executed")
    ist = hdr.index("Warp Stall Sampling (All Samples)")
    data = []
    for r in rows[2:]:
        try:
            data.append((int(r[ia], 16), int(r[iex]), int(r[ith]), int(r[ist])))
        except (ValueError, IndexError):
            pass
    base = data[0][0]
    tables = {}
    agg = defaultdict(lambda: [0, 0, 0])
    for ad, ex, th, st in data:
        f, ln = lm.get(ad - base, ("?", 0))
        key = f
        for d in ("csrc",):
            p = os.path.join(ROOT, "paper_2601_04860_b200", d, f)
            if os.path.exists(p):
                if p not in tables:
                    tables[p] = func_table(p)
                name = "?"
                for i, n in tables[p]:
                    if i <= ln:
                        name = n
                key = f"{f}:{name}"
        agg[key][0] += ex
        agg[key][1] += th
        agg[key][2] += st
    tw = sum(v[0] for v in agg.values()) or 1
    ts = sum(v[2] for v in agg.values()) or 1
    print(f"total warp instructions {tw/1e6:.1f} M, thread {sum(v[1] for v in agg.values())/1e6:.1f} M")
    for k, (ex, th, st) in sorted(agg.items(), key=lambda kv: -kv[1][0])[:a.top]:
        print(f"{k:40s} warp {ex/1e6:7.2f} M ({100*ex/tw:4.1f}%)  lanes {th/max(ex,1):5.1f}/32  "
              f"stall {100*st/ts:4.1f}%")


if __name__ == "__main__":
    main()
