"""Slab sharding host logic (paper_2601_04860_b200/sharding.py) on CPU.

The multi-process tests run two ranks over gloo on 127.0.0.1: rank 0 owns the
views, broadcasts them, every rank fuses its work-balanced axis-0 slab and the
occupancy slabs are all-gathered.  The per-slab fusion here is the CPU oracle
(test infrastructure standing in for the device kernel, which the GPU tests
cover); what is under test is the partition, the broadcast and the gather.
"""

import os
import socket
import types

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

import oracle
from paper_2601_04860_b200 import sharding
from tests import golden_io


def test_balanced_slabs_cover_and_balance():
    rng = np.random.default_rng(0)
    for g in (1, 2, 7, 64, 256):
        w = rng.random(g) * 10
        w[g // 3: g // 2] += 1000.0          # a mid-grid object, as in the scenes
        for n in (1, 2, 3, 4, 8):
            slabs = sharding.balanced_slabs(w, n)
            assert len(slabs) == n
            assert slabs[0][0] == 0 and slabs[-1][1] == g
            for (a, b), (c, d) in zip(slabs[:-1], slabs[1:]):
                assert b == c and a <= b
            if g >= n:
                assert all(b > a for a, b in slabs)
                bal = max(w[a:b].sum() for a, b in slabs)
                eq = max(w[a:b].sum() for a, b in sharding.equal_slabs(g, n))
                assert bal <= eq + 1e-9


def test_survey_imbalance_is_removed():
    """SURVEY.md section 7 hard part 6: equal 8-way slabs of sphere_on_plane at 256^3
    give max/mean gated work 2.52; balanced slabs must do far better."""
    import workloads
    from paper_2601_04860_b200.fusion import FusionParams
    dens, _o, _dx = workloads.density_grid(256)
    pv = FusionParams().as_vector()
    w = sharding.slice_weights(dens, pv, 32)
    w_np = sharding.slice_weights(dens.numpy(), pv, 32)
    assert np.allclose(w, w_np)
    gated = (dens.reshape(256, -1).numpy() >= 0.5).sum(1).astype(float)
    eq = [gated[a:b].sum() for a, b in sharding.equal_slabs(256, 8)]
    assert max(eq) / np.mean(eq) > 2.0
    bal = [w[a:b].sum() for a, b in sharding.balanced_slabs(w, 8)]
    assert max(bal) / np.mean(bal) < 1.15


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank, world, port, out):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        case = golden_io.scene_cases()["sop"]
        g = case.g
        nv, hm, wm = case.masks.shape
        names = ("masks", "dmins", "dmaxs", "dexps", "nsamps")
        cams = np.concatenate([case.rots.reshape(nv, 9), case.poss, case.intr], axis=1)
        if rank == 0:
            planes = {k: torch.from_numpy(np.ascontiguousarray(getattr(case, k))) for k in names}
            cam_t = torch.from_numpy(cams)
        else:
            planes = {k: torch.zeros((nv, hm, wm), dtype=torch.int32 if k == "nsamps"
                                     else torch.float32) for k in names}
            cam_t = torch.zeros((nv, 18), dtype=torch.float64)
        views = types.SimpleNamespace(cams=cam_t, z_surface=None, raw_masks=None, **planes)
        sharding.broadcast_views(views, src=0)
        for k in names:
            assert np.array_equal(getattr(views, k).numpy(), getattr(case, k)), k
        assert np.array_equal(views.cams.numpy(), cams)
        slabs = sharding.balanced_slabs(
            sharding.slice_weights(case.density.reshape(g, g, g), case.pv, nv), world)
        lo, hi = sharding.slab_voxel_range(slabs[rank], g)
        packed = (views.cams.numpy()[:, :9].reshape(nv, 3, 3), views.cams.numpy()[:, 9:12],
                  views.cams.numpy()[:, 12:18], views.masks.numpy(), views.dmins.numpy(),
                  views.dmaxs.numpy(), views.dexps.numpy(), views.nsamps.numpy(),
                  (views.nsamps.numpy() > 0).astype(np.uint8))
        r = oracle.fuse_packed(g, case.origin, case.dx, case.density, packed, case.pv, case.bc,
                               case.bh, case.unb, vox_range=(lo, hi))
        occ_slab = torch.from_numpy((r["p"][lo:hi] >= 0.5).astype(np.uint8))
        occ = sharding.gather_occupancy(occ_slab, slabs, g, rank)
        probs = sharding.gather_slab_values(torch.from_numpy(r["p"][lo:hi].copy()), slabs, g, rank)
        out[rank] = (occ.numpy().copy(), probs.numpy().copy(), slabs)
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 3])
def test_slab_sharded_fusion_gloo(world):
    case = golden_io.scene_cases()["sop"]
    manager = mp.Manager()
    out = manager.dict()
    mp.spawn(_worker, args=(world, _free_port(), out), nprocs=world, join=True)
    full = case.p
    for rank in range(world):
        occ, probs, slabs = out[rank]
        assert np.array_equal(occ.astype(bool), full >= 0.5)
        assert np.array_equal(probs, full)
        assert slabs[0][0] == 0 and slabs[-1][1] == case.g
