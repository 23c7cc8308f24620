"""A/B timing of library variants on the bench step (device-resident, L2 flushed).

    DIVAS_LIB=_variants/x.so python tools/ab_step.py --config C3 --iters 30

Prints one JSON line: refine / fuse ms (mean, min) of the bench step (windowed
records + fuse with the threshold fused) and a digest of the outputs (p bytes,
occupancy, votes) so variants can be checked for bit-identical results.
"""
import argparse
import hashlib
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="C3")
    ap.add_argument("--iters", type=int, default=30)
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
    g = wl.g
    probs = torch.empty(g ** 3, dtype=torch.float64, device=dev)
    occ = torch.empty(g ** 3, dtype=torch.uint8, device=dev)
    flush = torch.empty(256 << 20, dtype=torch.uint8, device=dev)
    roi = sharding.slab_view_rois(wl.density, params.as_vector(), g, wl.origin, wl.dx,
                                  pack_cameras(wl.cams), [tuple(wl.shape[1:])] * wl.nv)
    cap = fuser.capacity(wl.density, 0, g ** 3)
    ws = None
    bands = None
    tr, tf = [], []
    for i in range(args.iters + 5):
        flush.zero_()
        e = [torch.cuda.Event(enable_timing=True) for _ in range(3)]
        e[0].record()
        _m, bands = refine_bands_device(dv.raw_masks, dv.z_surface, dv.nsamps, dv.dexps, params,
                                        wl.dx, aux=bands, planar=False, roi=roi)
        e[1].record()
        out = fuser.run(wl.density, dv, probs=probs, occ=occ, workspace=ws, aux=bands,
                        max_gated=cap)
        ws = out["workspace"]
        e[2].record()
        torch.cuda.synchronize()
        if i >= 5:
            tr.append(e[0].elapsed_time(e[1]))
            tf.append(e[1].elapsed_time(e[2]))
    st = fuser.run(wl.density, dv, stats=True, occ=True, aux=bands, max_gated=cap)
    torch.cuda.synchronize()
    h = hashlib.sha256()
    for k in ("probs", "occ", "n_thick", "n_thin", "sw", "smw", "st"):
        h.update(st[k].cpu().numpy().tobytes())
    same = bool(torch.equal(st["probs"], probs) and torch.equal(st["occ"], occ))
    print(json.dumps({"lib": os.path.basename(_native.LIB_PATH), "config": args.config,
                      "refine_ms": sum(tr) / len(tr), "fuse_ms": sum(tf) / len(tf),
                      "fuse_min_ms": min(tf), "digest": h.hexdigest()[:16],
                      "votes": int((st["n_thick"] + st["n_thin"]).sum().item()),
                      "step_equals_stats_run": same}))


if __name__ == "__main__":
    main()
