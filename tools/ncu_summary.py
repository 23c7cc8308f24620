"""Summarise ncu outputs: launch lists (CSV) and --set full reports.

    python tools/ncu_summary.py launches gpurun_out/launches.csv [regex]
    python tools/ncu_summary.py report gpurun_out/prof.ncu-rep [--sass]
"""
import csv
import io
import re
import subprocess
import sys
from collections import defaultdict

KEYS = ["Duration", "Registers Per Thread", "Theoretical Occupancy", "Achieved Occupancy",
        "DRAM Throughput", "Memory Throughput", "L1/TEX Hit Rate", "L2 Hit Rate",
        "Issue Slots Busy", "Executed Ipc Active", "Warp Cycles Per Issued Instruction",
        "Avg. Active Threads Per Warp", "Branch Efficiency", "Executed Instructions"]


def launches(path, pat="divas"):
    rows = [r for r in csv.reader(l for l in open(path) if not l.startswith("=="))]
    hdr = rows[0]
    ki, vi, ui = hdr.index("Kernel Name"), hdr.index("Metric Value"), hdr.index("Metric Unit")
    agg = defaultdict(list)
    for r in rows[1:]:
        if re.search(pat, r[ki]):
            name = re.sub(r"\(.*", "", r[ki]).replace("void ", "")
            v = float(r[vi].replace(",", ""))
            scale = {"nsecond": 1e-3, "ns": 1e-3, "usecond": 1.0, "us": 1.0,
                     "msecond": 1e3, "ms": 1e3}.get(r[ui], 1.0)
            agg[name].append(v * scale)
    tot = sum(sum(v) for v in agg.values())
    for k, v in sorted(agg.items(), key=lambda kv: -sum(kv[1])):
        print(f"{k:45s} n={len(v):3d} mean={sum(v)/len(v):10.1f} us  share={100*sum(v)/tot:5.1f}%")


def report(path, sass=False):
    out = subprocess.run(["ncu", "-i", path, "--page", "details"], capture_output=True,
                         text=True).stdout
    for line in out.splitlines():
        s = line.strip()
        if ", Context " in s:                       # a kernel's section header
            print("== " + re.sub(r"\(.*?\)\s*\(", "(", s.split(", Context ")[0], count=1))
        elif any(s.startswith(k) for k in KEYS):
            print(s)
    raw = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True,
                         text=True).stdout
    rows = list(csv.reader(io.StringIO(raw)))
    if len(rows) > 2:
        hdr, vals = rows[0], rows[2]
        for k in ("dram__bytes_read.sum", "dram__bytes_write.sum", "lts__t_sector_hit_rate.pct",
                  "smsp__issue_active.avg.pct_of_peak_sustained_active", "gpu__time_duration.sum"):
            if k in hdr:
                print(f"{k} = {vals[hdr.index(k)]} {rows[1][hdr.index(k)]}")
    if sass:
        src = subprocess.run(["ncu", "-i", path, "--page", "source", "--csv", "--print-source",
                              "sass"], capture_output=True, text=True).stdout
        rows = list(csv.reader(io.StringIO(src)))
        hdr = rows[1]
        ia, isrc = hdr.index("Address"), hdr.index("Source")
        iex, ist = hdr.index("Instructions Executed"), hdr.index("Warp Stall Sampling (All Samples)")
        data = []
        for r in rows[2:]:
            try:
                data.append((int(r[ia], 16), int(r[iex]), int(r[ist]), r[isrc].strip()))
            except (ValueError, IndexError):
                pass
        base = data[0][0]
        b = defaultdict(lambda: [0, 0, ""])
        for a, ex, st, s in data:
            k = (a - base) // 0x400
            b[k][0] += ex
            b[k][1] += st
            b[k][2] = b[k][2] or s[:50]
        tot = sum(v[0] for v in b.values()) or 1
        tst = sum(v[1] for v in b.values()) or 1
        for k in sorted(b):
            if b[k][0] > 0.01 * tot or b[k][1] > 0.01 * tst:
                print(f"{hex(k * 0x400):>8s} instr {100*b[k][0]/tot:5.1f}%  stalls {100*b[k][1]/tst:5.1f}%  {b[k][2]}")


if __name__ == "__main__":
    if sys.argv[1] == "launches":
        launches(sys.argv[2], sys.argv[3] if len(sys.argv) > 3 else "divas")
    else:
        report(sys.argv[2], "--sass" in sys.argv)
