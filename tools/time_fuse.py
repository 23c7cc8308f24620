"""Quick device timing of refine / fuse for A/B experiments (not the bench).

    DIVAS_LIB=_variants/x.so python tools/time_fuse.py --config C3 --iters 20
"""
import argparse
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="C3")
    ap.add_argument("--iters", type=int, default=20)
    ap.add_argument("--bands", type=int, default=1)
    args = ap.parse_args()
    import torch
    import workloads
    from paper_2601_04860_b200 import _native
    from paper_2601_04860_b200.fusion import DeviceViews, FusionParams, Fuser, pack_cameras
    from paper_2601_04860_b200.segmenter import refine_bands_device, refine_masks_device
    dev = torch.device("cuda", 0)
    wl = workloads.make(args.config, device=dev, source=os.environ.get("DIVAS_INPUTS", "marcher"))
    dv = DeviceViews(torch.from_numpy(pack_cameras(wl.cams)).to(dev), torch.empty_like(wl.raw_masks),
                     wl.dmins, wl.dmaxs, wl.dexps, wl.nsamps, z_surface=wl.z_surface,
                     raw_masks=wl.raw_masks)
    grid = type("G", (), {"resolution": wl.g, "origin": wl.origin, "voxel_size": lambda s=None: wl.dx})()
    fuser = Fuser(grid, FusionParams())
    probs = torch.empty(wl.g ** 3, dtype=torch.float64, device=dev)
    flush = torch.empty(256 << 20, dtype=torch.uint8, device=dev)
    ws = None
    bands = None
    tr, tf = [], []
    for i in range(args.iters + 3):
        flush.zero_()
        e = [torch.cuda.Event(enable_timing=True) for _ in range(3)]
        e[0].record()
        if args.bands:
            _o, bands = refine_bands_device(dv.raw_masks, dv.z_surface, dv.nsamps, dv.dexps,
                                            FusionParams(), wl.dx, out=dv.masks, aux=bands)
        else:
            refine_masks_device(dv.raw_masks, dv.z_surface, dv.nsamps, out=dv.masks)
        e[1].record()
        out = fuser.run(wl.density, dv, probs=probs, occ=True, workspace=ws,
                        aux=bands if args.bands else None)
        ws = out["workspace"]
        e[2].record()
        torch.cuda.synchronize()
        if i >= 3:
            tr.append(e[0].elapsed_time(e[1]))
            tf.append(e[1].elapsed_time(e[2]))
    nz = int((probs != 0).sum().item())
    print(json.dumps({"lib": os.path.basename(_native.LIB_PATH), "config": args.config,
                      "refine_ms": sum(tr) / len(tr), "fuse_ms": sum(tf) / len(tf),
                      "fuse_min_ms": min(tf), "bands": args.bands, "nonzero": nz,
                      "psum": float(probs.sum().item())}))


if __name__ == "__main__":
    main()
