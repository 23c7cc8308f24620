"""Run a few device-resident fusion steps of a config (for ncu / launch lists)."""
import argparse
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="C3")
    ap.add_argument("--steps", type=int, default=3)
    ap.add_argument("--windows", default="on", choices=["on", "off"])
    args = ap.parse_args()
    import torch
    import workloads
    from paper_2601_04860_b200.fusion import DeviceViews, FusionParams, Fuser, pack_cameras
    from paper_2601_04860_b200.segmenter import refine_bands_device
    dev = torch.device("cuda", 0)
    wl = workloads.make(args.config, device=dev, source=os.environ.get("DIVAS_INPUTS", "marcher"))
    dv = DeviceViews(torch.from_numpy(pack_cameras(wl.cams)).to(dev), torch.empty_like(wl.raw_masks),
                     wl.dmins, wl.dmaxs, wl.dexps, wl.nsamps, z_surface=wl.z_surface,
                     raw_masks=wl.raw_masks)
    grid = type("G", (), {"resolution": wl.g, "origin": wl.origin, "voxel_size": lambda s=None: wl.dx})()
    fuser = Fuser(grid, FusionParams())
    probs = torch.empty(wl.g ** 3, dtype=torch.float64, device=dev)
    ws = None
    bands = None
    params = FusionParams()
    roi = None
    if args.windows == "on":
        from paper_2601_04860_b200 import sharding
        roi = sharding.slab_view_rois(wl.density, params.as_vector(), wl.g, wl.origin, wl.dx,
                                      pack_cameras(wl.cams), [tuple(wl.shape[1:])] * wl.nv)
    cap = fuser.capacity(wl.density, 0, wl.g ** 3)
    occ = torch.empty(wl.g ** 3, dtype=torch.uint8, device=dev)
    for _ in range(args.steps):      # the bench step: refine+records (windows), fuse
        _m, bands = refine_bands_device(dv.raw_masks, dv.z_surface, dv.nsamps, dv.dexps, params,
                                        wl.dx, aux=bands, planar=False, roi=roi)
        out = fuser.run(wl.density, dv, probs=probs, occ=occ, workspace=ws, aux=bands,
                        max_gated=cap)
        ws = out["workspace"]
    torch.cuda.synchronize()
    print("gated", int(Fuser.gated_count(out).item()))


if __name__ == "__main__":
    main()
