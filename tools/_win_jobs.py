"""The C3 window jobs of refine_and_fuse: sizes, and gather vs copy-engine
time per chunk in isolation (pinned sources)."""
import os, sys, time
sys.path.insert(0, os.getcwd())
import numpy as np, torch
import workloads
from paper_2601_04860_b200 import (ConfidenceMask, DensityGrid, VoxelGrid, ViewGeometry,
                                   refine_and_fuse, FusionParams, fusion, _native)
from paper_2601_04860_b200.geometry import Camera
dev = torch.device("cuda", 0)
wl = workloads.make("C3", device=dev, source="marcher")
def pinned(t):
    p = torch.empty(t.shape, dtype=t.dtype, pin_memory=True); p.copy_(t); return p.numpy()
pl = {k: pinned(getattr(wl, k)) for k in ("raw_masks", "z_surface", "dmins", "dmaxs", "dexps", "nsamps")}
grid = VoxelGrid(wl.g, workloads.GRID_HALF, wl.origin)
dens = DensityGrid(grid, pinned(wl.density).reshape(wl.g, wl.g, wl.g))
views = []
for v, c in enumerate(wl.cams):
    cam = Camera(c.fx, c.fy, c.cx, c.cy, c.width, c.height, c.world_from_camera)
    vg = ViewGeometry(cam, None, pl["dmins"][v], pl["dmaxs"][v], pl["dexps"][v], pl["nsamps"][v], pl["z_surface"][v])
    views.append((vg, ConfidenceMask(pl["raw_masks"][v])))
rec = []
orig = fusion._upload_windows
def spy(lib, jobs, stream):
    rec.append(list(jobs)); return orig(lib, jobs, stream)
fusion._upload_windows = spy
refine_and_fuse(grid, dens, views, FusionParams())
torch.cuda.synchronize()
lib = _native.lib()
s = torch.cuda.current_stream()
h = _native.stream_handle(s)
for ci, jobs in enumerate(rec):
    wb = [j[4] for j in jobs]; rows = [j[5] for j in jobs]
    by = sum(j[4] * j[5] for j in jobs)
    arr = (_native.Copy2D * len(jobs))(*[_native.Copy2D(*j) for j in jobs])
    def g():
        lib.divas_gather2d_h2d(arr, len(jobs), h)
    def c():
        for j in jobs:
            lib.divas_copy2d_h2d(j[1], j[3], j[0], j[2], j[4], j[5], h)
    out = []
    for fn in (g, c):
        fn(); torch.cuda.synchronize()
        e0 = torch.cuda.Event(enable_timing=True); e1 = torch.cuda.Event(enable_timing=True)
        e0.record(); [fn() for _ in range(5)]; e1.record(); torch.cuda.synchronize()
        out.append(e0.elapsed_time(e1) / 5)
    print(f"chunk {ci}: {len(jobs)} jobs {by/1e6:.2f} MB width_bytes {min(wb)}..{max(wb)} rows {min(rows)}..{max(rows)}"
          f"  gather {out[0]:.3f} ms ({by/out[0]/1e6:.1f} GB/s)  copy2d {out[1]:.3f} ms ({by/out[1]/1e6:.1f} GB/s)")
