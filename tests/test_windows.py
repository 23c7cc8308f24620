"""Per-view windows around the projected gated region (host logic, CPU)."""

import numpy as np
import pytest

from tests import golden_io
from tests.gpu_cases import cams_array


def _case():
    import torch
    case = golden_io.scene_cases()["sop"]
    return case, torch.from_numpy(case.density.reshape(-1).copy())


def test_view_windows_validation():
    from paper_2601_04860_b200.segmenter import ViewWindows
    w = ViewWindows([[0, 8, 15, 23], [8, 0, 8, 7]], "cpu")
    assert (w.max_w, w.max_h, w.nv) == (16, 16, 2)
    assert w.fraction(24, 16) == pytest.approx((16 * 16 + 1 * 8) / (2 * 24 * 16))
    with pytest.raises(ValueError):
        ViewWindows([[3, 0, 10, 10]], "cpu")            # x0 off the tile grid
    with pytest.raises(ValueError):
        ViewWindows([[8, 0, 7, 10]], "cpu")             # empty


def test_gated_bbox_matches_numpy():
    from paper_2601_04860_b200 import sharding
    case, dens = _case()
    g = case.g
    d = case.density.reshape(g, g, g).astype(np.float64)
    m = (d >= case.pv[4]) | ((case.pv[13] != 0) & (d >= case.pv[5]))
    ix, iy, iz = np.nonzero(m)
    assert sharding.gated_bbox(dens, case.pv, g) == \
        ((ix.min(), iy.min(), iz.min()), (ix.max(), iy.max(), iz.max()))
    lo, hi = sharding.slab_voxel_range((g // 2, g), g)
    sel = ix >= g // 2
    assert sharding.gated_bbox(dens, case.pv, g, (lo, hi)) == \
        ((ix[sel].min(), iy[sel].min(), iz[sel].min()), (ix[sel].max(), iy[sel].max(), iz[sel].max()))


@pytest.mark.parametrize("nslabs", [1, 3])
def test_windows_contain_every_footprint(nslabs):
    """Every pixel the fusion of a slab can read -- each gated voxel's centre
    pixel with its 4 neighbours and its corner box (fusion.py:170-192,
    :306-341, restated in numpy) -- lies inside that view's window."""
    from paper_2601_04860_b200 import sharding
    case, dens = _case()
    g, dx = case.g, case.dx
    cams = cams_array(case)
    sizes = [(int(h), int(w)) for w, h in case.intr[:, 4:6]]
    d = case.density.reshape(-1).astype(np.float64)
    gated = np.nonzero((d >= case.pv[4]) | ((case.pv[13] != 0) & (d >= case.pv[5])))[0]
    for slab in sharding.equal_slabs(g, nslabs):
        lo, hi = sharding.slab_voxel_range(slab, g)
        roi = sharding.slab_view_rois(dens, case.pv, g, case.origin, dx, cams, sizes, (lo, hi))
        vox = gated[(gated >= lo) & (gated < hi)]
        ix, rem = np.divmod(vox, g * g)
        iy, iz = np.divmod(rem, g)
        ctr = np.asarray(case.origin) + (np.stack([ix, iy, iz], 1) + 0.5) * dx
        for v, c in enumerate(cams):
            R, p = c[:9].reshape(3, 3), c[9:12]
            fx, fy, cx, cy, w, h = c[12:18]
            x0, y0, x1, y1 = roi.host[v]
            pts = [ctr] + [ctr + 0.5 * dx * np.array([sx, sy, sz])
                           for sx in (-1, 1) for sy in (-1, 1) for sz in (-1, 1)]
            for q in pts:
                rel = q - p
                dep = -(rel @ R[:, 2])
                ok = dep > 0
                u = (fx * ((rel @ R[:, 0])[ok] / dep[ok]) + cx) / w
                vv = (cy - fy * ((rel @ R[:, 1])[ok] / dep[ok])) / h
                px, py = np.floor(u * w), np.floor(vv * h)
                inside = (px >= 0) & (px < w) & (py >= 0) & (py < h)
                assert (px[inside] - 1 >= x0).all() or x0 == 0
                assert (px[inside] + 1 <= x1).all() or x1 == w - 1
                assert (py[inside] - 1 >= y0).all() or y0 == 0
                assert (py[inside] + 1 <= y1).all() or y1 == h - 1
