"""project_grid_overlay of the fused C3 grid onto a centroid-zoom view (for ncu)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def main():
    import torch
    import workloads
    from paper_2601_04860_b200 import VoxelGrid
    from paper_2601_04860_b200.fusion import (DeviceViews, FusionParams, Fuser, pack_cameras,
                                              project_grid_overlay_device)
    from paper_2601_04860_b200.geometry import Camera
    from paper_2601_04860_b200.segmenter import refine_bands_device
    dev = torch.device("cuda", 0)
    wl = workloads.make("C3", device=dev, source="marcher")
    dv = DeviceViews(torch.from_numpy(pack_cameras(wl.cams)).to(dev), torch.empty_like(wl.raw_masks),
                     wl.dmins, wl.dmaxs, wl.dexps, wl.nsamps, z_surface=wl.z_surface,
                     raw_masks=wl.raw_masks)
    params = FusionParams()
    _m, aux = refine_bands_device(dv.raw_masks, dv.z_surface, dv.nsamps, dv.dexps, params, wl.dx,
                                  out=dv.masks)
    grid = VoxelGrid(wl.g, workloads.GRID_HALF, wl.origin)
    probs = Fuser(grid, params).run(wl.density, dv, aux=aux)["probs"]
    i = wl.nv - 1
    c = wl.cams[i]
    cam = Camera(c.fx, c.fy, c.cx, c.cy, c.width, c.height, c.world_from_camera)
    for _ in range(3):
        out = project_grid_overlay_device(probs, grid, cam, wl.dmins[i], wl.dmaxs[i], wl.nsamps[i])
    torch.cuda.synchronize()
    print("overlay pixels on", int(out.sum().item()))


if __name__ == "__main__":
    main()
