"""Workload statistics against the survey's measurements on the reference's
fixture: gated voxels, vote totals, n_samples mix.

    python tools/input_stats.py [--config C1] [--inputs marcher|analytic]
"""

from __future__ import annotations

import argparse
import json
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    import torch
    import workloads
    from paper_2601_04860_b200.fusion import DeviceViews, Fuser, FusionParams
    from paper_2601_04860_b200.geometry import VoxelGrid
    from paper_2601_04860_b200.segmenter import refine_masks_device

    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="C1")
    ap.add_argument("--inputs", default="marcher")
    a = ap.parse_args()
    dev = torch.device("cuda", 0)
    wl = workloads.make(a.config, device=dev, source=a.inputs)
    from paper_2601_04860_b200.fusion import pack_cameras
    refined = refine_masks_device(wl.raw_masks, wl.z_surface, wl.nsamps)
    cams_t = torch.from_numpy(pack_cameras(wl.cams)).to(dev)
    dv = DeviceViews(cams_t, refined, wl.dmins, wl.dmaxs, wl.dexps, wl.nsamps)
    grid = VoxelGrid(wl.g, workloads.GRID_HALF, wl.origin)
    f = Fuser(grid, FusionParams())
    out = f.run(wl.density, dv, occ=True, stats=True)
    torch.cuda.synchronize()
    n = wl.nsamps
    res = {"config": a.config, "inputs": a.inputs,
           "gated": int(Fuser.gated_count(out).item()),
           "sum_n_thick": int(out["n_thick"].sum()), "sum_n_thin": int(out["n_thin"].sum()),
           "occupied": int(out["occ"].sum()),
           "n_samples_hist": {int(k): int(v) for k, v in zip(*np.unique(n.cpu().numpy(),
                                                                          return_counts=True))}}
    # views whose supporting pixels (refined mask > 0.5, n > 0) do not share one n
    sup = (refined > 0.5) & (n > 0)
    varied = 0
    for v in range(n.shape[0]):
        vals = torch.unique(n[v][sup[v]])
        varied += int(vals.numel() > 1)
    res["views_varied_tau"] = varied
    res["supporting_px_n_gt1"] = int(((n > 1) & sup).sum())
    print(json.dumps(res))


if __name__ == "__main__":
    main()
