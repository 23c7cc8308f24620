import sys, os, time; sys.path.insert(0, os.getcwd())
import numpy as np, torch
import workloads
from paper_2601_04860_b200 import (ConfidenceMask, DensityGrid, VoxelGrid, ViewGeometry, refine_and_fuse, FusionParams)
from paper_2601_04860_b200.geometry import Camera
import paper_2601_04860_b200.staging as stg_mod
dev = torch.device("cuda", 0)
wl = workloads.make("C3", device=dev, source="marcher")
import os
PIN = os.environ.get("PIN") == "1"
def host(t):
    if PIN:
        p = torch.empty(t.shape, dtype=t.dtype, pin_memory=True); p.copy_(t); return p.numpy()
    return t.cpu().numpy().copy()
planes = {k: host(getattr(wl, k)) for k in ("raw_masks", "z_surface", "dmins", "dmaxs", "dexps", "nsamps")}
grid = VoxelGrid(wl.g, workloads.GRID_HALF, wl.origin)
dens = DensityGrid(grid, host(wl.density).reshape(wl.g, wl.g, wl.g))
views = []
for v, c in enumerate(wl.cams):
    cam = Camera(c.fx, c.fy, c.cx, c.cy, c.width, c.height, c.world_from_camera)
    vg = ViewGeometry(cam, None, planes["dmins"][v], planes["dmaxs"][v], planes["dexps"][v], planes["nsamps"][v], planes["z_surface"][v])
    views.append((vg, ConfidenceMask(planes["raw_masks"][v])))
params = FusionParams()
# instrument Stager methods
S = stg_mod.Stager
orig_flush = S.flush
log = []
def flush(self):
    t0 = time.perf_counter(); orig_flush(self); log.append(("flush", time.perf_counter() - t0, self.bytes))
S.flush = flush
for rep in range(3):
    log.clear()
    torch.cuda.synchronize(); t0 = time.perf_counter()
    og, ref = refine_and_fuse(grid, dens, views, params)
    t = time.perf_counter() - t0
    print(f"rep {rep}: {t*1e3:.1f} ms; flushes:", [(n, round(d*1e3, 2), b >> 20) for n, d, b in log])
import cProfile, pstats
pr = cProfile.Profile(); pr.enable()
og, ref = refine_and_fuse(grid, dens, views, params)
pr.disable()
pstats.Stats(pr).sort_stats("cumulative").print_stats(18)
