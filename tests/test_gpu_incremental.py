"""Incremental session fusion (C4) == full recompute == the CPU oracle's
refine + fuse of the resulting view set, bit for bit (the reference session
recomputes everything on every update, session.py:212-215)."""

import numpy as np
import pytest

from tests import golden_io
from tests.gpu_cases import reference_objects

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def scene():
    from paper_2601_04860_b200 import ConfidenceMask, FusionParams
    raw, z, _refined = golden_io.scene_raw()
    case = golden_io.scene_cases()["sop"]
    grid, dens, views, bounds = reference_objects(case)
    for v, (vg, _m) in enumerate(views):
        vg.z_surface = z[v].copy()
    pairs = [(vg, ConfidenceMask(raw[v])) for v, (vg, _m) in enumerate(views)]
    params = FusionParams(*[float(x) for x in case.pv[:13]], enable_thin=bool(case.pv[13]))
    return grid, dens, pairs, params, bounds


def _oracle(grid, dens, pairs, params, bounds):
    """The CPU oracle on the same (view, raw mask) set: refine_mask then fuse
    of the refined set -- the reference session's full recompute
    (session.py:204-215)."""
    import oracle
    from paper_2601_04860_b200 import ConfidenceMask
    refined = [(vg, ConfidenceMask(oracle.refine(np.asarray(m.values, np.float32), vg.z_surface,
                                                 vg.n_samples), refined=True))
               for vg, m in pairs]
    return oracle.fuse(grid, dens, refined, params, bounds)["p"]


def _full(grid, dens, pairs, params, bounds):
    from paper_2601_04860_b200 import refine_and_fuse
    og, _m = refine_and_fuse(grid, dens, pairs, params, bounds=bounds, return_refined=False)
    return og.probs


def test_add_views_one_by_one(scene):
    from paper_2601_04860_b200 import FusionSession
    grid, dens, pairs, params, bounds = scene
    h, w = pairs[0][0].z_surface.shape
    s = FusionSession(grid, dens, params, (h, w), bounds=bounds, max_views=40)
    for k, (vg, m) in enumerate(pairs):
        assert s.add_view(vg, m) == k
        got = s.occupancy_grid().probs
        assert np.array_equal(got, _full(grid, dens, pairs[:k + 1], params, bounds)), k
        assert np.array_equal(got, _oracle(grid, dens, pairs[:k + 1], params, bounds)), k


def test_replace_mask_equals_recompute(scene):
    from paper_2601_04860_b200 import ConfidenceMask, FusionSession
    grid, dens, pairs, params, bounds = scene
    h, w = pairs[0][0].z_surface.shape
    s = FusionSession(grid, dens, params, (h, w), bounds=bounds, max_views=8)
    s.add_views(pairs[:5])
    rng = np.random.default_rng(4)
    cur = list(pairs[:5])
    for it in range(6):
        i = int(rng.integers(0, 5))
        new = ConfidenceMask(np.clip(cur[i][1].values * rng.uniform(0.3, 1.5), 0, 1))
        s.replace_mask(i, new)
        cur[i] = (cur[i][0], new)
        assert np.array_equal(s.occupancy_grid().probs, _full(grid, dens, cur, params, bounds))
        assert np.array_equal(s.occupancy_grid().probs, _oracle(grid, dens, cur, params, bounds))
    s.refuse()
    assert np.array_equal(s.occupancy_grid().probs, _full(grid, dens, cur, params, bounds))
    with pytest.raises(ValueError):
        s.add_views(pairs[:4])          # capacity 8 exceeded
    with pytest.raises(IndexError):
        s.replace_mask(7, cur[0][1])


def test_mixed_resolution_session():
    from paper_2601_04860_b200 import ConfidenceMask, FusionParams, FusionSession
    case = golden_io.scene_cases()["mixed"]
    grid, dens, views, bounds = reference_objects(case)
    pairs = [(vg, ConfidenceMask(m.values)) for vg, m in views]
    params = FusionParams(*[float(x) for x in case.pv[:13]], enable_thin=bool(case.pv[13]))
    hm = max(vg.z_surface.shape[0] for vg, _ in pairs)
    wm = max(vg.z_surface.shape[1] for vg, _ in pairs)
    s = FusionSession(grid, dens, params, (hm, wm), bounds=bounds, max_views=4)
    s.add_view(*pairs[2])               # the small view first, then the larger ones
    s.add_views(pairs[:2])
    order = [pairs[2], pairs[0], pairs[1]]
    assert np.array_equal(s.occupancy_grid().probs, _full(grid, dens, order, params, bounds))


@pytest.mark.parametrize("graph", [True, False])
def test_replace_mask_device_graph_replay(scene, graph):
    """Device-side replacements, replayed from captured CUDA graphs (a view's
    graph is reused across updates with new masks) or launched eagerly, give
    the full recompute's bits; adding a view invalidates the graphs."""
    import torch
    from paper_2601_04860_b200 import ConfidenceMask, FusionSession
    grid, dens, pairs, params, bounds = scene
    h, w = pairs[0][0].z_surface.shape
    s = FusionSession(grid, dens, params, (h, w), bounds=bounds, max_views=8)
    s.add_views(pairs[:4])
    rng = np.random.default_rng(11)
    cur = list(pairs[:4])
    for it in range(8):
        i = it % 3                                  # views 0..2 reuse their graphs
        vals = np.clip(cur[i][1].values * rng.uniform(0.3, 1.5), 0, 1).astype(np.float32)
        s.replace_mask_device(i, torch.from_numpy(vals).to(s.dev), graph=graph)
        cur[i] = (cur[i][0], ConfidenceMask(vals))
        assert np.array_equal(s.occupancy_grid().probs, _full(grid, dens, cur, params, bounds))
        assert np.array_equal(s.occupancy_grid().probs, _oracle(grid, dens, cur, params, bounds))
    assert (len(s._graphs) == 3) == graph
    s.add_views(pairs[4:5])
    cur.append(pairs[4])
    assert not s._graphs
    vals = np.clip(cur[0][1].values * 0.7, 0, 1).astype(np.float32)
    s.replace_mask_device(0, torch.from_numpy(vals).to(s.dev), graph=graph)
    cur[0] = (cur[0][0], ConfidenceMask(vals))
    assert np.array_equal(s.occupancy_grid().probs, _full(grid, dens, cur, params, bounds))
