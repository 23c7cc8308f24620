"""Per-stage pair counters of fuse_pairs (experiment build with DIVAS_STATS=1).

    python -m paper_2601_04860_b200.build --variant _variants/stats.so -D DIVAS_STATS=1
    DIVAS_LIB=_variants/stats.so python tools/pair_stats.py --config C3
"""
import argparse
import ctypes
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

NAMES = ["pairs", "in_frustum", "valid_px", "thick_try", "thick_depth_ok", "thick_vote",
         "thin_gated", "band_tiles", "scan_items", "scan_pixels", "unsure_recounts",
         "thin_votes", "thick_exact_fallback", "corner_exact_fallback", "centre_uncertain",
         "band_too_wide", "items_mmax_below_accept", "pixels_mmax_below_accept",
         "items_zero_support", "pixels_zero_support", "items_full_support", "pixels_full_support",
         "items_64px_or_more", "pixels_64px_or_more"]


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="C3")
    args = ap.parse_args()
    import torch
    import workloads
    from paper_2601_04860_b200 import _native
    from paper_2601_04860_b200.fusion import DeviceViews, FusionParams, Fuser, pack_cameras
    from paper_2601_04860_b200.segmenter import refine_bands_device
    dev = torch.device("cuda", 0)
    wl = workloads.make(args.config, device=dev, source=os.environ.get("DIVAS_INPUTS", "marcher"))
    dv = DeviceViews(torch.from_numpy(pack_cameras(wl.cams)).to(dev), torch.empty_like(wl.raw_masks),
                     wl.dmins, wl.dmaxs, wl.dexps, wl.nsamps, z_surface=wl.z_surface,
                     raw_masks=wl.raw_masks)
    grid = type("G", (), {"resolution": wl.g, "origin": wl.origin, "voxel_size": lambda s=None: wl.dx})()
    fuser = Fuser(grid, FusionParams())
    lib = _native.lib()
    f = lib.divas_debug_pair_stats
    buf = (ctypes.c_ulonglong * 24)()
    _o, aux = refine_bands_device(dv.raw_masks, dv.z_surface, dv.nsamps, dv.dexps, FusionParams(),
                                  wl.dx, out=dv.masks)
    f(buf, 1)
    fuser.run(wl.density, dv, occ=True, aux=aux)
    f(buf, 1)
    print(json.dumps({"config": args.config, **{n: int(v) for n, v in zip(NAMES, buf)}}))


if __name__ == "__main__":
    main()
