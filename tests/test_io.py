"""Wire formats (io.py of the reference): byte-identical files."""

import io

import numpy as np
import pytest

from tests import golden_io
from tests.golden_io import GOLDEN


def _gold():
    return dict(np.load(GOLDEN + "/scene.npz"))


def test_fmap_bytes_and_roundtrip():
    from paper_2601_04860_b200.io import read_fmap, write_fmap
    d = _gold()
    case = golden_io.scene_cases()["sop"]
    h, w = int(case.intr[0, 5]), int(case.intr[0, 4])
    buf = io.BytesIO()
    write_fmap(buf, case.dexps[0, :h, :w])
    assert buf.getvalue() == d["sop_fmap_bytes"].tobytes()
    buf.seek(0)
    assert np.array_equal(read_fmap(buf), case.dexps[0, :h, :w])
    rgb = np.random.default_rng(0).random((5, 4, 3)).astype(np.float32)
    b2 = io.BytesIO()
    write_fmap(b2, rgb)
    b2.seek(0)
    assert np.array_equal(read_fmap(b2), rgb)
    with pytest.raises(ValueError):
        write_fmap(io.BytesIO(), np.zeros(3))


@pytest.mark.gpu
def test_vgrid_bytes_and_roundtrip():
    from paper_2601_04860_b200 import OccupancyGrid
    from paper_2601_04860_b200.io import read_vgrid, write_vgrid
    from tests.gpu_cases import reference_objects
    d = _gold()
    case = golden_io.scene_cases()["sop"]
    grid, _dens, _views, _b = reference_objects(case)
    og = OccupancyGrid(grid, case.p)
    buf = io.BytesIO()
    write_vgrid(buf, og, unbounded=False)
    assert buf.getvalue() == d["sop_vgrid_bytes"].tobytes()
    buf.seek(0)
    og2, unb = read_vgrid(buf)
    assert not unb
    assert np.array_equal(og2.probs, og.probs.astype(np.float32).astype(np.float64))
    # odd sizes exercise the tile edges
    import torch
    from paper_2601_04860_b200.io import vgrid_payload_device
    for g in (1, 5, 33, 70):
        p = np.random.default_rng(g).random((g, g, g))
        got = vgrid_payload_device(torch.from_numpy(p).cuda(), g).cpu().numpy()
        assert np.array_equal(got, p.astype("<f4").transpose(2, 1, 0).ravel())
