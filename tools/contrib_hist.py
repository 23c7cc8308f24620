"""Per-voxel contribution counts (n_thick, n_thin) over the gated voxels of a
config: what the value-sorted reduction (fuse_reduce) has to sort."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def main():
    import numpy as np
    import torch
    import workloads
    from paper_2601_04860_b200.fusion import DeviceViews, FusionParams, Fuser, pack_cameras
    cfg = sys.argv[1] if len(sys.argv) > 1 else "C5"
    dev = torch.device("cuda", 0)
    wl = workloads.make(cfg, device=dev, source="marcher")
    dv = DeviceViews(torch.from_numpy(pack_cameras(wl.cams)).to(dev), wl.raw_masks.clone(),
                     wl.dmins, wl.dmaxs, wl.dexps, wl.nsamps)
    from paper_2601_04860_b200.segmenter import refine_masks_device
    refine_masks_device(wl.raw_masks, wl.z_surface, wl.nsamps, out=dv.masks)
    grid = type("G", (), {"resolution": wl.g, "origin": wl.origin, "voxel_size": lambda s=None: wl.dx})()
    out = Fuser(grid, FusionParams()).run(wl.density, dv, stats=True)
    idx = Fuser.gated_voxels(out)
    nt = out["n_thick"].reshape(-1)[idx].cpu().numpy()
    nn = out["n_thin"].reshape(-1)[idx].cpu().numpy()
    for name, a in (("thick", nt), ("thin", nn), ("both", nt + nn)):
        q = np.percentile(a, [50, 90, 99, 100])
        print(f"{cfg} {name}: mean {a.mean():.1f} p50 {q[0]:.0f} p90 {q[1]:.0f} p99 {q[2]:.0f} max {q[3]:.0f}"
              f"  sum n^2/4 {np.sum(a.astype(np.float64) ** 2) / 4 / 1e6:.1f} M")
    print(f"{cfg} gated {idx.numel()}")


if __name__ == "__main__":
    main()
