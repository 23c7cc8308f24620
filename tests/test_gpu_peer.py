"""The slab all-gather fused into the fusion's stores (``occ_peers``).

Every "rank" fuses its axis-0 slab and stores the slab's occupancy bytes into
every listed buffer; after all slabs, each buffer must equal the occupancy of
the full fusion bit for bit.  On one GPU the buffers are plain device tensors
(the pointer table is what a multi-GPU run fills with NVLink peer mappings),
plus one run through real symmetric memory in a world-size-1 process group.
"""

import numpy as np
import pytest

from tests import golden_io
from tests.gpu_cases import bounds_ns, device_views, grid_ns

pytestmark = pytest.mark.gpu


def _setup(name="sop"):
    import torch
    from paper_2601_04860_b200.fusion import Fuser
    case = golden_io.scene_cases()[name]
    dev = torch.device("cuda", 0)
    dv = device_views(case, dev)
    fuser = Fuser(grid_ns(case), case.pv, bounds_ns(case))
    dens = torch.from_numpy(case.density.reshape(-1)).to(dev)
    full = fuser.run(dens, dv, occ=True)
    return case, dev, dv, fuser, dens, full["occ"].clone()


@pytest.mark.parametrize("world", [1, 2, 3])
def test_peer_occupancy_stores_equal_full(world):
    import torch
    from paper_2601_04860_b200 import sharding
    case, dev, dv, fuser, dens, occ_full = _setup()
    g = case.g
    slabs = sharding.equal_slabs(g, world)
    bufs = [torch.full((g ** 3,), 7, dtype=torch.uint8, device=dev) for _ in range(world)]
    table = torch.tensor([b.data_ptr() for b in bufs], dtype=torch.int64, device=dev)
    for r in range(world):
        lo, hi = sharding.slab_voxel_range(slabs[r], g)
        fuser.run(dens, dv, vox_range=(lo, hi), occ=None, occ_peers=(table.data_ptr(), world))
    torch.cuda.synchronize()
    for b in bufs:
        assert torch.equal(b, occ_full)


def test_peer_occupancy_symmetric_memory_world1():
    import os
    import socket

    import torch
    import torch.distributed as dist
    from paper_2601_04860_b200 import sharding
    case, dev, dv, fuser, dens, occ_full = _setup()
    with socket.socket() as sk:
        sk.bind(("127.0.0.1", 0))
        port = sk.getsockname()[1]
    os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
    dist.init_process_group("nccl", init_method=f"tcp://127.0.0.1:{port}", rank=0,
                            world_size=1, device_id=dev)
    try:
        peer = sharding.PeerOccupancy(case.g ** 3, dev)
        for b in peer.bufs:
            b.fill_(9)
        # two steps: each writes its own buffer (double-buffered, no WAR race)
        for step in range(2):
            first = peer.buf
            fuser.run(dens, dv, occ=None, occ_peers=peer.peers)
            got = peer.barrier()
            torch.cuda.synchronize()
            assert got.data_ptr() == first.data_ptr()
            assert peer.buf.data_ptr() != first.data_ptr()
            assert peer.world == 1
            assert torch.equal(got, occ_full)
    finally:
        dist.destroy_process_group()


def test_peer_occupancy_unaligned_slab():
    """Slab bounds that are not multiples of 4 voxels take the scalar stores."""
    import torch
    case, dev, dv, fuser, dens, occ_full = _setup()
    n = case.g ** 3
    cuts = [0, n // 3 + 1, 2 * n // 3 + 2, n]
    buf = torch.zeros(n, dtype=torch.uint8, device=dev)
    table = torch.tensor([buf.data_ptr()], dtype=torch.int64, device=dev)
    for lo, hi in zip(cuts[:-1], cuts[1:]):
        fuser.run(dens, dv, vox_range=(lo, hi), occ=None, occ_peers=(table.data_ptr(), 1))
    torch.cuda.synchronize()
    assert torch.equal(buf, occ_full)
    assert int(np.count_nonzero(occ_full.cpu().numpy())) > 0


def test_peer_put_blocks():
    """divas_peer_put stores one block into every listed buffer at an offset."""
    import torch
    from paper_2601_04860_b200 import _native
    dev = torch.device("cuda", 0)
    bufs = [torch.zeros(3 * 1000 + 7, dtype=torch.uint8, device=dev) for _ in range(3)]
    table = torch.tensor([b.data_ptr() for b in bufs], dtype=torch.int64, device=dev)
    for r, nbytes in enumerate((1000, 1003, 17)):
        src = torch.randint(0, 255, (nbytes,), dtype=torch.uint8, device=dev)
        off = r * 1000 + (r == 2)
        _native.check(_native.lib().divas_peer_put(src.data_ptr(), nbytes, table.data_ptr(), 3,
                                                   off, _native.stream_handle()), "peer_put")
        torch.cuda.synchronize()
        for b in bufs:
            assert torch.equal(b[off:off + nbytes], src)


def test_peer_gather_world1():
    import os
    import socket

    import torch
    import torch.distributed as dist
    from paper_2601_04860_b200 import sharding
    dev = torch.device("cuda", 0)
    with socket.socket() as sk:
        sk.bind(("127.0.0.1", 0))
        port = sk.getsockname()[1]
    os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
    dist.init_process_group("nccl", init_method=f"tcp://127.0.0.1:{port}", rank=0,
                            world_size=1, device_id=dev)
    try:
        pg = sharding.PeerGather((5, 4), torch.int32, dev)
        src = torch.arange(20, dtype=torch.int32, device=dev).reshape(5, 4)
        out = pg.gather(src)
        torch.cuda.synchronize()
        assert torch.equal(out[0], src)
    finally:
        dist.destroy_process_group()
