"""Time the fixture producers on the device: render_view of a camera rig of
the ``sphere_on_plane`` scene with the reference's render config (384
samples per ray) and bake_density_grid, plus the CPU oracle on a sample.

    python tools/time_render.py [--config C3] [--reps 5]
"""

from __future__ import annotations

import argparse
import json
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    import torch
    import oracle
    import workloads
    from paper_2601_04860_b200.geometry import VoxelGrid
    from paper_2601_04860_b200.render import render_views_device
    from paper_2601_04860_b200.scene import bake_density_device
    from tests import golden_io

    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="C3")
    ap.add_argument("--reps", type=int, default=5)
    a = ap.parse_args()
    c = workloads.CONFIGS[a.config]
    sc = golden_io.render_scene("sop")
    sc.bounds = golden_io.Bounds(np.array([-4.9, -4.4, -4.9]), np.array([4.9, 5.5, 4.9]), False)
    cams = workloads.cameras(c["views"], c["n"], c["w"], c["h"])
    cfg = golden_io.GoldCfg(384, 0.4, 12.5, 0.75, 1e-4)
    grid = VoxelGrid(c["g"], workloads.GRID_HALF,
                     np.asarray(workloads.CENTER) - workloads.GRID_HALF)
    ev = lambda: torch.cuda.Event(enable_timing=True)  # noqa: E731
    out = {"config": a.config, "views": len(cams), "w": c["w"], "h": c["h"], "g": c["g"]}
    for _ in range(2):
        o = render_views_device(sc, cams, cfg, unsure=True)
        bake_density_device(sc, grid)
    torch.cuda.synchronize()
    ts, tb = [], []
    for _ in range(a.reps):
        e0, e1, e2 = ev(), ev(), ev()
        e0.record()
        o = render_views_device(sc, cams, cfg, unsure=True)
        e1.record()
        bake_density_device(sc, grid)
        e2.record()
        torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1))
        tb.append(e1.elapsed_time(e2))
    npx = len(cams) * c["w"] * c["h"]
    out["render_ms"] = float(np.median(ts))
    out["render_rays_per_s"] = npx / (out["render_ms"] * 1e-3)
    out["unsure_px"] = int(o["unsure"].sum())
    out["mean_samples_marched"] = None
    out["bake_ms"] = float(np.median(tb))
    out["bake_voxels_per_s"] = c["g"] ** 3 / (out["bake_ms"] * 1e-3)
    # CPU oracle on one camera row band (all threads), extrapolated
    cam = cams[0]
    band = max(1, c["h"] // 16)

    class Sub:
        pass
    s = Sub()
    s.rotation, s.position = cam.rotation, cam.position
    s.fx, s.fy, s.cx, s.cy, s.width, s.height = cam.fx, cam.fy, cam.cx, cam.cy, cam.width, band
    t0 = time.perf_counter()
    oracle.render(sc.arrays(), s, cfg)
    dt = time.perf_counter() - t0
    out["cpu_oracle_rays_per_s"] = cam.width * band / dt
    out["cpu_threads"] = oracle.max_threads()
    print(json.dumps(out))


if __name__ == "__main__":
    main()
