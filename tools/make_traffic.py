"""profiles/ncu_traffic.json from an ncu DRAM-bytes launch list of the bench
step (bench.py reads it for roofline.traffic).

    python tools/make_traffic.py gpurun_out/prof/traffic_C3.csv C3 "<source note>"
"""
import csv
import json
import os
import re
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
FUSE = ("gate_tiles", "gate_scan", "gate_emit", "fuse_pairs", "fuse_reduce<32>")
REFINE = ("refine_minmax<4>", "band_pass<4, 1>")


def main():
    path, config, note = sys.argv[1], sys.argv[2], sys.argv[3]
    rows = list(csv.reader(l for l in open(path) if not l.startswith("==")))
    hdr = rows[0]
    ki, mi, vi = hdr.index("Kernel Name"), hdr.index("Metric Name"), hdr.index("Metric Value")
    idx = hdr.index("ID")
    per = {}
    for r in rows[1:]:
        name = re.sub(r"\(.*", "", r[ki]).replace("void ", "").replace("divas::", "")
        per.setdefault(name, {}).setdefault(int(r[idx]), 0.0)
        per[name][int(r[idx])] += float(r[vi].replace(",", ""))
    last = {k: v[max(v)] for k, v in per.items()}          # last launch per kernel
    out_path = os.path.join(ROOT, "profiles", "ncu_traffic.json")
    data = json.load(open(out_path)) if os.path.exists(out_path) else {}
    data["_source"] = note
    data[config] = {"fuse": sum(last.get(k, 0.0) for k in FUSE),
                    "refine": sum(last.get(k, 0.0) for k in REFINE), "per_kernel": last}
    json.dump(data, open(out_path, "w"), indent=1)
    print(json.dumps(data[config]))


if __name__ == "__main__":
    main()
