"""The split step plan of the bench (and of any caller overlapping the dense
zero fill with the pair kernel): GATE|GATE_KEEP|CLEAR_ALL, ZERO, PAIRS, REDUCE
on poisoned output buffers give the one-call fusion bit for bit, on two
streams as the bench runs them; GATE_KEEP leaves the outputs untouched."""

import numpy as np
import pytest

from tests import golden_io
from tests.gpu_cases import bounds_ns, device_views, grid_ns

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("scene", ["sop", "small"])
@pytest.mark.parametrize("vox_range", [None, "slab"])
def test_split_steps_equal_full(scene, vox_range):
    import torch
    from paper_2601_04860_b200 import _native
    from paper_2601_04860_b200.fusion import Fuser
    case = golden_io.scene_cases()[scene]
    dev = torch.device("cuda", 0)
    dv = device_views(case, dev)
    fuser = Fuser(grid_ns(case), case.pv, bounds_ns(case))
    g = case.g
    dens = torch.from_numpy(case.density.reshape(-1)).to(dev)
    lo, hi = (0, g ** 3) if vox_range is None else ((g // 3) * g * g, (2 * g // 3 + 1) * g * g)
    ref = fuser.run(dens, dv, stats=True, occ=True, vox_range=(lo, hi))
    probs = torch.full((g ** 3,), 7.0, dtype=torch.float64, device=dev)     # poison
    occ = torch.full((g ** 3,), 9, dtype=torch.uint8, device=dev)
    kw = dict(probs=probs, occ=occ, vox_range=(lo, hi), max_gated=fuser.capacity(dens, lo, hi))
    side = torch.cuda.Stream(dev)
    o = fuser.run(dens, dv, steps=_native.STEP_GATE | _native.STEP_GATE_KEEP |
                  _native.STEP_CLEAR_ALL, **kw)
    ws = o["workspace"]
    torch.cuda.synchronize()
    # the gate left the outputs alone
    assert float(probs[lo:hi].min()) == 7.0 and int(occ[lo:hi].min()) == 9
    side.wait_stream(torch.cuda.current_stream())
    with torch.cuda.stream(side):
        fuser.run(dens, dv, workspace=ws, steps=_native.STEP_ZERO, stream=side, **kw)
    fuser.run(dens, dv, workspace=ws, steps=_native.STEP_PAIRS, view_range=(0, dv.nv), **kw)
    torch.cuda.current_stream().wait_stream(side)
    fuser.run(dens, dv, workspace=ws, steps=_native.STEP_REDUCE, **kw)
    torch.cuda.synchronize()
    assert torch.equal(probs[lo:hi], ref["probs"][lo:hi])
    assert torch.equal(occ[lo:hi], ref["occ"][lo:hi])
    # outside the range nothing was written
    assert bool((probs[:lo] == 7.0).all()) and bool((probs[hi:] == 7.0).all())
    assert bool((occ[:lo] == 9).all()) and bool((occ[hi:] == 9).all())


def test_zero_step_unaligned_ranges():
    """ZERO over ranges that do not start or end on a 16-voxel group."""
    import torch
    from paper_2601_04860_b200 import _native
    from paper_2601_04860_b200.fusion import Fuser
    case = golden_io.scene_cases()["sop"]
    dev = torch.device("cuda", 0)
    dv = device_views(case, dev)
    fuser = Fuser(grid_ns(case), case.pv, bounds_ns(case))
    g = case.g
    dens = torch.from_numpy(case.density.reshape(-1)).to(dev)
    for lo, hi in [(3, 7), (5, 40), (17, g ** 3 - 3), (0, 1), (g ** 3 - 1, g ** 3)]:
        probs = torch.full((g ** 3,), 7.0, dtype=torch.float64, device=dev)
        occ = torch.full((g ** 3,), 9, dtype=torch.uint8, device=dev)
        fuser.run(dens, dv, probs=probs, occ=occ, vox_range=(int(lo), int(hi)), max_gated=1,
                  steps=_native.STEP_ZERO)
        torch.cuda.synchronize()
        p, o = probs.cpu().numpy(), occ.cpu().numpy()
        assert np.all(p[lo:hi] == 0.0) and np.all(o[lo:hi] == 0)
        assert np.all(p[:lo] == 7.0) and np.all(p[hi:] == 7.0)
        assert np.all(o[:lo] == 9) and np.all(o[hi:] == 9)
