"""Where the end-to-end update time goes (host timers, synchronised phases).

    python tools/e2e_breakdown.py --config C3
"""
import argparse
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="C3")
    ap.add_argument("--iters", type=int, default=5)
    args = ap.parse_args()
    import numpy as np
    import torch
    import workloads
    from paper_2601_04860_b200 import FusionParams, refine_and_fuse
    from paper_2601_04860_b200.fusion import (Fuser, _sparse_probs_to_host, _upload_planes,
                                              pack_cameras, DeviceViews)
    from paper_2601_04860_b200._device import as_device
    from paper_2601_04860_b200.segmenter import refine_bands_device
    import bench
    dev = torch.device("cuda", 0)
    wl = workloads.make(args.config, device=dev, source=os.environ.get("DIVAS_INPUTS", "marcher"))
    params = FusionParams()

    class A:
        e2e_steps = args.iters
    # full API
    r = bench.run_e2e(A, wl, params, dev)
    out = {"e2e_ms": r["ms_per_step"]}
    # raw pinned H2D bandwidth
    n = 512 << 20
    h = torch.empty(n, dtype=torch.uint8, pin_memory=True)
    d = torch.empty(n, dtype=torch.uint8, device=dev)
    for _ in range(2):
        d.copy_(h, non_blocking=True)
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(3):
        d.copy_(h, non_blocking=True)
    torch.cuda.synchronize()
    out["h2d_GBps"] = 3 * n / (time.perf_counter() - t0) / 1e9
    t0 = time.perf_counter()
    for _ in range(3):
        h.copy_(d, non_blocking=True)
    torch.cuda.synchronize()
    out["d2h_GBps"] = 3 * n / (time.perf_counter() - t0) / 1e9
    # phases with the same inputs
    from paper_2601_04860_b200 import ConfidenceMask, DensityGrid, VoxelGrid, ViewGeometry
    from paper_2601_04860_b200.geometry import Camera

    def pinned(t):
        p = torch.empty(t.shape, dtype=t.dtype, pin_memory=True)
        p.copy_(t)
        return p.numpy()
    planes = {k: pinned(getattr(wl, k)) for k in
              ("raw_masks", "z_surface", "dmins", "dmaxs", "dexps", "nsamps")}
    grid = VoxelGrid(wl.g, workloads.GRID_HALF, wl.origin)
    dens = DensityGrid(grid, pinned(wl.density).reshape(wl.g, wl.g, wl.g))
    views = []
    for v, c in enumerate(wl.cams):
        cam = Camera(c.fx, c.fy, c.cx, c.cy, c.width, c.height, c.world_from_camera)
        vg = ViewGeometry(cam, None, planes["dmins"][v], planes["dmaxs"][v], planes["dexps"][v],
                          planes["nsamps"][v], planes["z_surface"][v])
        views.append((vg, ConfidenceMask(planes["raw_masks"][v])))
    ph = {}
    for it in range(args.iters + 1):
        T = {}
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        vgs = [vg for vg, _m in views]
        pl, sizes, cams = _upload_planes(vgs, [m for _vg, m in views], dev,
                                         ("raw", "z", "dmins", "dmaxs", "dexps", "nsamps"))
        dd = as_device(dens.values, np.float32, dev)
        torch.cuda.synchronize()
        T["upload"] = time.perf_counter() - t0
        t0 = time.perf_counter()
        fuser = Fuser(grid, params)
        refined, aux = refine_bands_device(pl["raw"], pl["z"], pl["nsamps"], pl["dexps"],
                                           fuser.pv, fuser.dx, planar=True)
        dv = DeviceViews(torch.from_numpy(pack_cameras(cams)).to(dev), refined, pl["dmins"],
                         pl["dmaxs"], pl["dexps"], pl["nsamps"], sizes=sizes)
        o = fuser.run(dd, dv, aux=aux)
        torch.cuda.synchronize()
        T["compute"] = time.perf_counter() - t0
        t0 = time.perf_counter()
        host = torch.empty(refined.shape, dtype=torch.float32, pin_memory=True)
        host.copy_(refined, non_blocking=True)
        torch.cuda.synchronize()
        T["refined_d2h"] = time.perf_counter() - t0
        t0 = time.perf_counter()
        probs = _sparse_probs_to_host(o, wl.g ** 3)
        T["probs_host"] = time.perf_counter() - t0
        t0 = time.perf_counter()
        hn = host.numpy()
        ms = [hn[i] for i in range(len(sizes))]
        T["wrap"] = time.perf_counter() - t0
        if it:
            for k, v in T.items():
                ph.setdefault(k, []).append(v * 1e3)
    out.update({k: float(np.median(v)) for k, v in ph.items()})
    print(json.dumps(out))


if __name__ == "__main__":
    main()
