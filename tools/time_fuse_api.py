"""The drop-in fuse() API at C3 from ordinary (pageable) numpy inputs, as a
reference caller hands them over: the refined masks and view maps of the
workload, b200.fuse(grid, density, views, params) -> host OccupancyGrid."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def main():
    import numpy as np
    import torch
    import workloads
    from paper_2601_04860_b200 import (ConfidenceMask, DensityGrid, FusionParams, VoxelGrid,
                                       ViewGeometry, fuse)
    from paper_2601_04860_b200.geometry import Camera
    from paper_2601_04860_b200.segmenter import refine_masks_device
    cfg = sys.argv[1] if len(sys.argv) > 1 else "C3"
    dev = torch.device("cuda", 0)
    wl = workloads.make(cfg, device=dev, source="marcher")
    refined = torch.empty_like(wl.raw_masks)
    refine_masks_device(wl.raw_masks, wl.z_surface, wl.nsamps, out=refined)
    host = lambda t: t.cpu().numpy().copy()            # noqa: E731  (pageable numpy)
    grid = VoxelGrid(wl.g, workloads.GRID_HALF, wl.origin)
    dens = DensityGrid(grid, host(wl.density).reshape(wl.g, wl.g, wl.g))
    views = []
    for v, c in enumerate(wl.cams):
        cam = Camera(c.fx, c.fy, c.cx, c.cy, c.width, c.height, c.world_from_camera)
        vg = ViewGeometry(cam, None, host(wl.dmins[v]), host(wl.dmaxs[v]), host(wl.dexps[v]),
                          host(wl.nsamps[v]), host(wl.z_surface[v]))
        m = ConfidenceMask.__new__(ConfidenceMask)
        m.values, m.refined = host(refined[v]), True
        views.append((vg, m))
    params = FusionParams()
    og = fuse(grid, dens, views, params)
    torch.cuda.synchronize()
    ts = []
    for _ in range(5):
        t0 = time.perf_counter()
        og = fuse(grid, dens, views, params)
        ts.append(1e3 * (time.perf_counter() - t0))
    print(f"{cfg} fuse() API from pageable numpy: median {np.median(ts):.2f} ms "
          f"({[round(t, 2) for t in ts]}), occupied {int((og.probs >= 0.5).sum())}")


if __name__ == "__main__":
    main()
