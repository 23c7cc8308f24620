"""profiles/ncu_traffic.json from an ncu launch list of the bench step
(dram__bytes_read/write.sum, gpu__time_duration.sum, smsp__inst_executed.sum;
tools/refresh_profiles.sh).  bench.py reads it for roofline.traffic (DRAM
bytes per launch of the dominant operator) and roofline.issue (warp
instructions per launch, for the issue-rate roofline).

    python tools/make_traffic.py gpurun_out/prof_r02/launches_C3.csv C3 "<source note>"
"""
import csv
import json
import os
import re
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
FUSE = ("gate_tiles", "gate_scan", "gate_emit", "tile_cull", "fuse_pairs", "fuse_reduce")
REFINE = ("refine_init", "refine_minmax", "band_init", "band_pass")


def group(name):
    base = re.sub(r"<.*", "", name)
    if any(base.startswith(k) for k in FUSE):
        return "fuse"
    if any(base.startswith(k) for k in REFINE):
        return "refine"
    return None


def main():
    path, config, note = sys.argv[1], sys.argv[2], sys.argv[3]
    rows = list(csv.reader(l for l in open(path) if not l.startswith("==")))
    hdr = rows[0]
    ki, mi, vi = hdr.index("Kernel Name"), hdr.index("Metric Name"), hdr.index("Metric Value")
    idx = hdr.index("ID")
    per = {}
    for r in rows[1:]:
        name = re.sub(r"\(.*", "", r[ki]).replace("void ", "").replace("divas::", "")
        launch = per.setdefault(name, {}).setdefault(int(r[idx]), {})
        launch[r[mi]] = float(r[vi].replace(",", ""))
    last = {k: v[max(v)] for k, v in per.items()}          # last launch per kernel
    out_path = os.path.join(ROOT, "profiles", "ncu_traffic.json")
    data = json.load(open(out_path)) if os.path.exists(out_path) else {}
    data["_source"] = note
    rec = {"per_kernel": {}}
    for g in ("fuse", "refine"):
        ks = [k for k in last if group(k) == g]
        rec[g] = sum(last[k].get("dram__bytes_read.sum", 0) + last[k].get("dram__bytes_write.sum", 0)
                     for k in ks)
        rec[g + "_inst"] = sum(last[k].get("smsp__inst_executed.sum", 0) for k in ks)
        rec[g + "_ns"] = sum(last[k].get("gpu__time_duration.sum", 0) for k in ks)
    for k, m in last.items():
        rec["per_kernel"][k] = {"dram_bytes": m.get("dram__bytes_read.sum", 0) +
                                m.get("dram__bytes_write.sum", 0),
                                "warp_inst": m.get("smsp__inst_executed.sum"),
                                "ns": m.get("gpu__time_duration.sum")}
    data[config] = rec
    json.dump(data, open(out_path, "w"), indent=1)
    print(json.dumps({k: v for k, v in rec.items() if k != "per_kernel"}))


if __name__ == "__main__":
    main()
