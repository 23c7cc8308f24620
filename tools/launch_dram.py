"""Summarise an ncu launch CSV with gpu__time_duration + dram bytes per kernel."""
import csv
import sys
from collections import defaultdict

rows = [r for r in csv.reader(l for l in open(sys.argv[1]) if not l.startswith('=='))]
h = rows[0]
ki, mi, vi, ui = h.index("Kernel Name"), h.index("Metric Name"), h.index("Metric Value"), h.index("Metric Unit")
d = defaultdict(lambda: defaultdict(list))
scale = {"ns": 1e-3, "nsecond": 1e-3, "us": 1.0, "usecond": 1.0, "msecond": 1e3, "byte": 1.0,
         "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}   # times -> us, sizes -> bytes
for r in rows[1:]:
    d[r[ki].split('(')[0]][r[mi]].append(float(r[vi].replace(',', '')) * scale.get(r[ui], 1.0))
for k, m in sorted(d.items(), key=lambda kv: -sum(kv[1]['gpu__time_duration.sum'])):
    n = len(m['gpu__time_duration.sum'])
    t = sum(m['gpu__time_duration.sum']) / n
    rb = sum(m['dram__bytes_read.sum']) / max(len(m['dram__bytes_read.sum']), 1)
    wb = sum(m['dram__bytes_write.sum']) / max(len(m['dram__bytes_write.sum']), 1)
    inst = m.get('smsp__inst_executed.sum')
    ins = f"  {sum(inst) / len(inst) / 1e6:7.2f} M warp-inst" if inst else ""
    print(f"{k:32s} n={n:2d} {t:8.1f} us  read {rb/1e6:7.1f} MB  write {wb/1e6:7.1f} MB  "
          f"{(rb + wb) / (t * 1e3):6.0f} GB/s{ins}")
