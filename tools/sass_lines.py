"""Map ncu SASS hot spots to CUDA source lines via nvdisasm line info.

    python tools/sass_lines.py <ncu-rep> <kernel-substring> [<source .cu> ...]
"""
import csv
import io
import os
import re
import subprocess
import sys
import tempfile
from collections import defaultdict

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
LIB = os.environ.get("SASS_LIB") or os.path.join(ROOT, "paper_2601_04860_b200", "_lib", "libdivas_b200.so")


def line_map(kernel):
    tmp = tempfile.mkdtemp()
    subprocess.run(["cuobjdump", "-xelf", "all", LIB], cwd=tmp, capture_output=True)
    out = {}
    for f in os.listdir(tmp):
        dis = subprocess.run(["nvdisasm", "-g", "-c", os.path.join(tmp, f)], capture_output=True,
                             text=True).stdout
        infn, cur = False, None
        for line in dis.splitlines():
            if line.startswith("//----") and ".text." in line:
                infn = kernel in line
                continue
            if not infn:
                continue
            m = re.search(r'//## File "([^"]+)", line (\d+)', line)
            if m:
                cur = (os.path.basename(m.group(1)), int(m.group(2)))
                continue
            m = re.match(r"\s+/\*([0-9a-f]{4,})\*/", line)
            if m and cur:
                out[int(m.group(1), 16)] = cur
    return out


def main():
    rep, kernel = sys.argv[1], sys.argv[2]
    lm = line_map(kernel)
    src = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"],
                         capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(src)))
    hdr = rows[1]
    ia, iex = hdr.index("Address"), hdr.index("Instructions Executed")
    ist = hdr.index("Warp Stall Sampling (All Samples)")
    data = []
    for r in rows[2:]:
        try:
            data.append((int(r[ia], 16), int(r[iex]), int(r[ist])))
        except (ValueError, IndexError):
            pass
    base = data[0][0]
    agg = defaultdict(lambda: [0, 0])
    for a, ex, st in data:
        key = lm.get(a - base, ("?", 0))
        agg[key][0] += ex
        agg[key][1] += st
    tot = sum(v[0] for v in agg.values()) or 1
    tst = sum(v[1] for v in agg.values()) or 1
    srcs = {}
    for (f, ln), (ex, st) in sorted(agg.items(), key=lambda kv: -kv[1][0])[:int(os.environ.get("TOP", "40"))]:
        path = os.path.join(ROOT, "paper_2601_04860_b200", "csrc", f)
        if f not in srcs and os.path.exists(path):
            srcs[f] = open(path).read().splitlines()
        text = srcs.get(f, [""] * (ln + 1))[ln - 1].strip() if ln else ""
        print(f"{100*ex/tot:5.1f}% instr {100*st/tst:5.1f}% stall  {f}:{ln:<5d} {text[:80]}")


if __name__ == "__main__":
    main()
