"""Views-sharding on one GPU: the per-rank step sequence (GATE, broadcast of
the gated list, PAIRS on a view block, contribution exchange, REDUCE),
simulated rank by rank, reproduces the full fusion bit for bit."""

import numpy as np
import pytest

from tests import golden_io
from tests.gpu_cases import bounds_ns, device_views, grid_ns

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("world", [2, 3, 8])
def test_view_sharded_steps_equal_full(world):
    import torch
    from paper_2601_04860_b200 import _native
    from paper_2601_04860_b200.fusion import Fuser
    from paper_2601_04860_b200.sharding import ViewShardPlan
    case = golden_io.scene_cases()["sop"]
    dev = torch.device("cuda", 0)
    dv = device_views(case, dev)
    fuser = Fuser(grid_ns(case), case.pv, bounds_ns(case))
    dens = torch.from_numpy(case.density.reshape(-1)).to(dev)
    full = fuser.run(dens, dv, stats=True)["probs"].clone()
    cap = fuser.capacity(dens, 0, case.g ** 3)
    plan = ViewShardPlan(dv.nv, world, cap, dv.hm, dv.wm)
    outs, wss = [], []
    for r in range(world):                      # GATE on every "rank"
        o = fuser.run(dens, dv, steps=_native.STEP_GATE, nv_cap=plan.nv_cap, max_gated=cap)
        outs.append(o)
        wss.append(o["workspace"])
    reg = plan.reg
    for r in range(1, world):                   # broadcast rank 0's gated list
        wss[r][:8].copy_(wss[0][:8])
        wss[r][reg["work"]: reg["work"] + 4 * cap].copy_(wss[0][reg["work"]: reg["work"] + 4 * cap])
    for r, (v0, v1) in enumerate(plan.blocks):  # PAIRS on the rank's block
        if v1 > v0:
            fuser.run(dens, dv, probs=outs[r]["probs"], workspace=wss[r], nv_cap=plan.nv_cap,
                      max_gated=cap, steps=_native.STEP_CLEAR_ALL | _native.STEP_PAIRS,
                      view_range=(v0, v1))
        else:
            fuser.run(dens, dv, probs=outs[r]["probs"], workspace=wss[r], nv_cap=plan.nv_cap,
                      max_gated=cap, steps=_native.STEP_CLEAR_ALL)
    rb = plan.rows * cap * 8                    # exchange (what all_gather / all_reduce do)
    for k in ("w", "mw", "t"):
        for r in range(world):
            blk = slice(reg[k] + r * rb, reg[k] + (r + 1) * rb)
            for q in range(world):
                if q != r:
                    wss[q][blk].copy_(wss[r][blk])
    bits = [w[reg["bits_thick"]: reg["w"]].view(torch.int32) for w in wss]
    tot = torch.stack(bits).sum(0)
    for b in bits:
        b.copy_(tot)
    for r in range(world):                      # REDUCE everywhere
        fuser.run(dens, dv, probs=outs[r]["probs"], workspace=wss[r], nv_cap=plan.nv_cap,
                  max_gated=cap, steps=_native.STEP_REDUCE)
        assert torch.equal(outs[r]["probs"], full), r
