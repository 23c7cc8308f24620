"""Parts of the pinned e2e update, timed alone (H2D / D2H link rates, the host
zero fill of the result grid) -- to see what bounds refine_and_fuse."""
import os, sys, time
sys.path.insert(0, os.getcwd())
import numpy as np, torch
dev = torch.device("cuda", 0)
torch.cuda.init()
def t(fn, n=5):
    fn(); torch.cuda.synchronize()
    ts = []
    for _ in range(n):
        t0 = time.perf_counter(); fn(); torch.cuda.synchronize(); ts.append(time.perf_counter() - t0)
    return 1e3 * float(np.median(ts))
E2E_ONLY = os.environ.get("E2E_ONLY") == "1"
nb = 436 << 20 if not E2E_ONLY else 1 << 20
hp = torch.empty(nb, dtype=torch.uint8, pin_memory=True)
dd = torch.empty(nb, dtype=torch.uint8, device=dev)
print("h2d 436MB pinned ms", t(lambda: dd.copy_(hp, non_blocking=True)))
nb2 = 99 << 20
print("d2h 99MB pinned ms", t(lambda: hp[:nb2].copy_(dd[:nb2], non_blocking=True)))
s2 = torch.cuda.Stream()
def duplex():
    with torch.cuda.stream(s2):
        hp[nb - nb2:].copy_(dd[:nb2], non_blocking=True)
    dd[:nb - nb2].copy_(hp[:nb - nb2], non_blocking=True)
print("h2d 337MB || d2h 99MB ms", t(duplex))
g3 = 256 ** 3
print("zeroed host grid (134MB pinned alloc+zero) ms", t(lambda: torch.empty(g3, dtype=torch.float64, pin_memory=True).zero_()))
x = torch.empty(g3, dtype=torch.float64, pin_memory=True)
print("zero_ only ms", t(lambda: x.zero_()))
print("torch threads", torch.get_num_threads(), "cpus", os.cpu_count())

# one pinned refine_and_fuse under the torch profiler: the device timeline
import workloads
from paper_2601_04860_b200 import (ConfidenceMask, DensityGrid, VoxelGrid, ViewGeometry,
                                   refine_and_fuse, FusionParams)
from paper_2601_04860_b200.geometry import Camera
wl = workloads.make("C3", device=dev, source="marcher")
def pinned(t):
    if os.environ.get("PAGEABLE") == "1":
        return t.cpu().numpy().copy()
    p = torch.empty(t.shape, dtype=t.dtype, pin_memory=True); p.copy_(t); return p.numpy()
pl = {k: pinned(getattr(wl, k)) for k in ("raw_masks", "z_surface", "dmins", "dmaxs", "dexps", "nsamps")}
grid = VoxelGrid(wl.g, workloads.GRID_HALF, wl.origin)
dens = DensityGrid(grid, pinned(wl.density).reshape(wl.g, wl.g, wl.g))
views = []
for v, c in enumerate(wl.cams):
    cam = Camera(c.fx, c.fy, c.cx, c.cy, c.width, c.height, c.world_from_camera)
    vg = ViewGeometry(cam, None, pl["dmins"][v], pl["dmaxs"][v], pl["dexps"][v], pl["nsamps"][v], pl["z_surface"][v])
    views.append((vg, ConfidenceMask(pl["raw_masks"][v])))
params = FusionParams()
for _ in range(3):
    refine_and_fuse(grid, dens, views, params)
torch.cuda.synchronize()
ts = []
for _ in range(9):
    t0 = time.perf_counter(); r = refine_and_fuse(grid, dens, views, params); ts.append(time.perf_counter() - t0); r = None
print("e2e", "pageable" if os.environ.get("PAGEABLE") == "1" else "pinned", "ms",
      [round(1e3 * x, 2) for x in ts], os.environ.get("DIVAS_LIB", "cur"),
      os.environ.get("DIVAS_STAGE_THREADS", ""))
if E2E_ONLY:
    sys.exit(0)
from torch.profiler import profile, ProfilerActivity
with profile(activities=[ProfilerActivity.CPU, ProfilerActivity.CUDA]) as prof:
    t0 = time.perf_counter(); r = refine_and_fuse(grid, dens, views, params); torch.cuda.synchronize()
    print("profiled e2e ms", 1e3 * (time.perf_counter() - t0))
prof.export_chrome_trace("gpurun_out/e2e_trace.json")
import json
tr = json.load(open("gpurun_out/e2e_trace.json"))
ev = [e for e in tr["traceEvents"] if e.get("ph") == "X" and e.get("cat") in ("kernel", "gpu_memcpy", "gpu_memset", "cuda_runtime", "cpu_op", "python_function")]
t0 = min(e["ts"] for e in ev)
rows = sorted(((e["ts"] - t0) / 1e3, e["dur"] / 1e3, e["cat"], e.get("args", {}).get("stream", ""), e["name"][:60]) for e in ev if e["cat"] in ("kernel", "gpu_memcpy", "gpu_memset"))
for r_ in rows:
    print("%8.3f %7.3f %-10s s%-4s %s" % r_)
cpu = sorted(((e["ts"] - t0) / 1e3, e["dur"] / 1e3, e["name"][:70]) for e in ev if e["cat"] == "cuda_runtime" and e["dur"] > 200)
print("-- slow runtime calls (>0.2 ms)")
for r_ in cpu:
    print("%8.3f %7.3f %s" % r_)
