"""Fallback / skip counters of one bench-step fusion (DIVAS_FB_* of the C ABI).

    python tools/fallbacks.py --config C3
"""
import argparse
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="C3")
    args = ap.parse_args()
    import torch
    import workloads
    from paper_2601_04860_b200 import _native, sharding
    from paper_2601_04860_b200.fusion import DeviceViews, FusionParams, Fuser, pack_cameras
    from paper_2601_04860_b200.segmenter import refine_bands_device
    dev = torch.device("cuda", 0)
    wl = workloads.make(args.config, device=dev, source=os.environ.get("DIVAS_INPUTS", "marcher"))
    dv = DeviceViews(torch.from_numpy(pack_cameras(wl.cams)).to(dev), torch.empty_like(wl.raw_masks),
                     wl.dmins, wl.dmaxs, wl.dexps, wl.nsamps, z_surface=wl.z_surface,
                     raw_masks=wl.raw_masks)
    grid = type("G", (), {"resolution": wl.g, "origin": wl.origin, "voxel_size": lambda s=None: wl.dx})()
    params = FusionParams()
    fuser = Fuser(grid, params)
    roi = sharding.slab_view_rois(wl.density, params.as_vector(), wl.g, wl.origin, wl.dx,
                                  pack_cameras(wl.cams), [tuple(wl.shape[1:])] * wl.nv)
    _m, bands = refine_bands_device(dv.raw_masks, dv.z_surface, dv.nsamps, dv.dexps, params,
                                    wl.dx, planar=False, roi=roi)
    fb = torch.zeros(_native.NFALLBACK, dtype=torch.int64, device=dev)
    out = fuser.run(wl.density, dv, aux=bands, fallbacks=fb, stats=True)
    torch.cuda.synchronize()
    gated = int(Fuser.gated_count(out).item())
    tiles = -(-gated // 256) * wl.nv
    rec = {"config": args.config, "gated": gated, "pairs": gated * wl.nv, "pair_tiles": tiles,
           "votes_thick": int(out["n_thick"].sum().item()),
           "votes_thin": int(out["n_thin"].sum().item())}
    rec.update({k: int(v) for k, v in zip(_native.FALLBACKS, fb.cpu().tolist())})
    print(json.dumps(rec))


if __name__ == "__main__":
    main()
