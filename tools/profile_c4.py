"""A few C4 updates (re-refine + re-fuse one view of the fused C3 state) for ncu."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def main():
    import torch
    import workloads
    from paper_2601_04860_b200 import DensityGrid, FusionParams, FusionSession, VoxelGrid
    from paper_2601_04860_b200.fusion import pack_cameras
    dev = torch.device("cuda", 0)
    wl = workloads.make("C3", device=dev, source="marcher")
    nv, H, W = wl.shape
    grid = VoxelGrid(wl.g, workloads.GRID_HALF, wl.origin)
    dens = DensityGrid(grid, wl.density.cpu().numpy().reshape(wl.g, wl.g, wl.g))
    s = FusionSession(grid, dens, FusionParams(), (H, W), max_views=nv + 1, dev=dev)
    for name, src in (("raw", wl.raw_masks), ("z", wl.z_surface), ("dmins", wl.dmins),
                      ("dmaxs", wl.dmaxs), ("dexps", wl.dexps), ("nsamps", wl.nsamps)):
        getattr(s, name)[:nv].copy_(src)
    s.cams[:nv].copy_(torch.from_numpy(pack_cameras(wl.cams)))
    s.sizes = [(H, W)] * nv
    s.nv = nv
    s._refine(0, nv)
    s._fuse(0, nv)
    torch.cuda.synchronize()
    for k in range(6):
        s.replace_mask_device(k % nv, torch.roll(wl.raw_masks[k % nv], 1, 1).contiguous(),
                              graph=False)
    torch.cuda.synchronize()
    print("ok")


if __name__ == "__main__":
    main()
