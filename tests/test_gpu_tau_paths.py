"""The footprint scan's three record paths (bands.cuh, fuse.cu thin_item),
each forced on the golden sop scene through the refine+bands pass and
checked against the oracle:

* const   -- every supporting pixel has one tau: plane A alone;
* flagged -- a few supporting pixels differ from the base tau(n_min): plane A
             alone with the base tau, items meeting a flagged pixel recounted;
* planeB  -- many differ: plane A + plane B (per-pixel tau).
"""

import dataclasses

import numpy as np
import pytest

import oracle
from tests import golden_io
from tests.gpu_cases import bounds_ns, cams_array, grid_ns

pytestmark = pytest.mark.gpu


def _entries(bands, nv, hm, wm):
    """Each view's two trailing 16-byte entries (tau keys, counts, base tau):
    the per-view band block is divas_bands_size(1, hm, wm) bytes, tiles first."""
    from paper_2601_04860_b200 import _native
    stride = int(_native.lib().divas_bands_size(1, hm, wm)) // 16
    ntiles = stride - 2
    b = bands.view(np.uint32).reshape(nv, stride * 4)
    return b[:, ntiles * 4: ntiles * 4 + 8]


@pytest.mark.parametrize("mode", ["const", "flagged", "planeB"])
def test_scan_paths_match_oracle(mode):
    import torch
    from paper_2601_04860_b200.fusion import DeviceViews, Fuser
    from paper_2601_04860_b200.segmenter import refine_bands_device
    case = golden_io.scene_cases()["sop"]
    raw, z, refined = golden_io.scene_raw()
    n = case.nsamps.copy()
    sup = (refined > 0.5) & (n > 0)
    n[n > 0] = 2                                # base: n_min = 1 must exist somewhere
    n[sup] = 1
    rng = np.random.default_rng(3)
    idx = np.flatnonzero(sup)
    if mode == "flagged":
        n.reshape(-1)[rng.choice(idx, size=max(1, len(idx) // 200), replace=False)] = 3
    elif mode == "planeB":
        n.reshape(-1)[rng.choice(idx, size=len(idx) // 2, replace=False)] = 3
    dev = torch.device("cuda", 0)
    t = lambda a: torch.from_numpy(np.ascontiguousarray(a)).to(dev)  # noqa: E731
    out, aux = refine_bands_device(t(raw), t(z), t(n), t(case.dexps), case.pv, case.dx)
    assert np.array_equal(out.cpu().numpy(), refined)
    nv, hm, wm = raw.shape
    e = _entries(aux.bands.cpu().numpy(), nv, hm, wm)
    tk0, tk1, nflag, nsup = e[:, 0], e[:, 1], e[:, 2].astype(np.int64), e[:, 3].astype(np.int64)
    has = nsup > 0
    assert has.any()
    if mode == "const":
        assert np.all(tk0[has] == tk1[has]) and np.all(nflag == 0)
    elif mode == "flagged":
        varied = has & (tk0 < tk1)
        assert varied.any() and np.all(nflag[varied] * 32 <= nsup[varied])
    else:
        varied = has & (tk0 < tk1)
        assert varied.any() and np.all(nflag[varied] * 32 > nsup[varied])
    dv = DeviceViews(t(cams_array(case)), out, t(case.dmins), t(case.dmaxs), t(case.dexps), t(n))
    fuser = Fuser(grid_ns(case), case.pv, bounds_ns(case))
    dens = torch.from_numpy(case.density.reshape(-1)).to(dev)
    got = fuser.run(dens, dv, stats=True, occ=True, aux=aux)
    torch.cuda.synchronize()
    c2 = dataclasses.replace(case, masks=refined, nsamps=n)
    ref = oracle.fuse_packed(c2.g, c2.origin, c2.dx, c2.density, c2.packed,
                             c2.pv, c2.bc, c2.bh, c2.unb)
    assert np.array_equal(got["n_thick"].cpu().numpy(), ref["n_thick"])
    assert np.array_equal(got["n_thin"].cpu().numpy(), ref["n_thin"])
    assert np.array_equal(got["st"].cpu().numpy(), ref["st"])
    p = got["probs"].cpu().numpy()
    assert np.array_equal(p >= 0.5, ref["p"] >= 0.5)
    rel = np.abs(p - ref["p"]) / np.maximum(np.abs(ref["p"]), 1e-300)
    assert rel.max(initial=0.0) <= 1e-12
    assert int(ref["n_thin"].sum()) > 0
