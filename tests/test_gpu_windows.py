"""Scan records built only inside per-view windows (divas_refine_bands_roi).

The fusion of a slab reads no record or band outside the projection of the
slab's gated voxels: with everything outside the windows poisoned (all-ones
bytes: NaN records / bands), the fused probabilities and votes equal the
full fusion's bit for bit."""

import numpy as np
import pytest

from tests import golden_io
from tests.gpu_cases import bounds_ns, cams_array, device_views, grid_ns

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("name", ["sop", "mixed"])
@pytest.mark.parametrize("nslabs", [1, 2, 3])
def test_windowed_records_equal_full(name, nslabs):
    import torch
    from paper_2601_04860_b200 import sharding
    from paper_2601_04860_b200.fusion import Fuser
    from paper_2601_04860_b200.segmenter import ViewAux, refine_bands_device
    case = golden_io.scene_cases()[name]
    dev = torch.device("cuda", 0)
    dv = device_views(case, dev)
    raw = dv.masks.clone()                       # treated as raw masks, refined below
    z = dv.dexps.clone()
    fuser = Fuser(grid_ns(case), case.pv, bounds_ns(case))
    dens = torch.from_numpy(case.density.reshape(-1)).to(dev)
    nv, hm, wm = dv.nv, dv.hm, dv.wm
    _o, full_aux = refine_bands_device(raw, z, dv.nsamps, dv.dexps, case.pv, case.dx,
                                       planar=False)
    full = fuser.run(dens, dv, stats=True, aux=full_aux)
    sizes = [(int(h), int(w)) for w, h in case.intr[:, 4:6]]
    g = case.g
    for slab in sharding.equal_slabs(g, nslabs):
        lo, hi = sharding.slab_voxel_range(slab, g)
        roi = sharding.slab_view_rois(dens, case.pv, g, case.origin, case.dx, cams_array(case),
                                      sizes, vox_range=(lo, hi))
        aux = ViewAux.empty(nv, hm, wm, dev)
        aux.records.fill_(0xFF)
        aux.bands.fill_(0xFF)
        refine_bands_device(raw, z, dv.nsamps, dv.dexps, case.pv, case.dx, aux=aux,
                            planar=False, roi=roi)
        out = fuser.run(dens, dv, stats=True, aux=aux, vox_range=(lo, hi))
        for k in ("probs", "n_thick", "n_thin", "sw", "smw", "st"):
            assert torch.equal(out[k][lo:hi], full[k][lo:hi]), (slab, k)
        assert roi.fraction(hm, wm) <= 1.0


def test_windowed_planar_output_inside_windows():
    """Inside its window, the planar refined output equals the full refine."""
    import torch
    from paper_2601_04860_b200 import sharding
    from paper_2601_04860_b200.segmenter import refine_bands_device
    case = golden_io.scene_cases()["sop"]
    raw, zs, refined = golden_io.scene_raw()
    dev = torch.device("cuda", 0)
    t = lambda a: torch.from_numpy(np.ascontiguousarray(a)).to(dev)  # noqa: E731
    sizes = [(int(h), int(w)) for w, h in case.intr[:, 4:6]]
    dens = t(case.density.reshape(-1))
    roi = sharding.slab_view_rois(dens, case.pv, case.g, case.origin, case.dx, cams_array(case),
                                  sizes)
    out = torch.full(raw.shape, -7.0, dtype=torch.float32, device=dev)
    refine_bands_device(t(raw), t(zs), t(case.nsamps), t(case.dexps), case.pv, case.dx,
                        out=out, roi=roi)
    o = out.cpu().numpy()
    for v, (x0, y0, x1, y1) in enumerate(roi.host):
        assert np.array_equal(o[v, y0:y1 + 1, x0:x1 + 1], refined[v, y0:y1 + 1, x0:x1 + 1])


def test_minmax_keys_split_equal_full():
    """Min/max keys computed in view blocks (as ranks do) + the keys-based band
    pass == the one-call refine: refined masks, records and bands bit-exact."""
    import torch
    from paper_2601_04860_b200.segmenter import (ViewAux, refine_bands_device,
                                                 refine_minmax_device)
    case = golden_io.scene_cases()["sop"]
    raw, zs, refined = golden_io.scene_raw()
    dev = torch.device("cuda", 0)
    t = lambda a: torch.from_numpy(np.ascontiguousarray(a)).to(dev)  # noqa: E731
    m, z, n, d = t(raw), t(zs), t(case.nsamps), t(case.dexps)
    nv, hm, wm = m.shape
    out_a, aux_a = refine_bands_device(m, z, n, d, case.pv, case.dx)
    keys = torch.zeros((nv, 4), dtype=torch.int32, device=dev)
    cut = nv // 2
    refine_minmax_device(z[:cut], n[:cut], keys=keys[:cut])
    refine_minmax_device(z[cut:], n[cut:], keys=keys[cut:])
    aux_b = ViewAux.empty(nv, hm, wm, dev)
    out_b, _ = refine_bands_device(m, z, n, d, case.pv, case.dx, aux=aux_b, keys=keys)
    assert torch.equal(out_a, out_b)
    assert np.array_equal(out_b.cpu().numpy(), refined)
    assert _records_equal(aux_a.records, aux_b.records, nv, hm, wm)
    assert torch.equal(aux_a.bands, aux_b.bands)


def _records_equal(ra, rb, nv, hm, wm):
    """Plane A everywhere; plane B where it is defined (A holds a depth: B is
    written only at pixels that can support, bands.cuh)."""
    import torch
    a = ra.view(torch.float32).view(nv, 2, hm, wm, 2)
    b = rb.view(torch.float32).view(nv, 2, hm, wm, 2)
    ai, bi = a.view(torch.int32), b.view(torch.int32)
    if not torch.equal(ai[:, 0], bi[:, 0]):
        return False
    defined = ~torch.isnan(a[:, 0, :, :, 1])
    return torch.equal(ai[:, 1][defined], bi[:, 1][defined])
