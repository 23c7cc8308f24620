"""Per-pair public operations and the decision trace vs the reference's own
outputs (tests/golden/trace.npz, made by tests/golden/make_golden.py).

Stages, flags, pixel boxes and counts must match exactly; floats to 1e-12
relative (the depth weight goes through CUDA's exp vs glibc's)."""

import json
import math

import numpy as np
import pytest

from tests.golden_io import GOLDEN

pytestmark = pytest.mark.gpu
REL = 1e-12


@pytest.fixture(scope="module")
def gold():
    return dict(np.load(GOLDEN + "/trace.npz"))


def _views(d, prefix):
    from paper_2601_04860_b200 import Camera, ConfidenceMask, ViewGeometry
    out = []
    for i in range(int(d[f"{prefix}_nv"])):
        fx, fy, cx, cy, w, h = d[f"{prefix}_v{i}_intr"]
        cam = Camera(fx, fy, cx, cy, int(w), int(h), d[f"{prefix}_v{i}_w2c"])
        g = lambda k: d[f"{prefix}_v{i}_{k}"]  # noqa: E731
        vg = ViewGeometry(cam, None, g("d_min"), g("d_max"), g("d_exp"), g("n_samples"),
                          g("z_surface"))
        out.append((vg, ConfidenceMask(g("mask"), refined=True)))
    return out


def _same(a, b, path=""):
    if isinstance(a, dict):
        assert a.keys() == b.keys(), path
        for k in a:
            _same(a[k], b[k], f"{path}.{k}")
    elif isinstance(a, list):
        assert len(a) == len(b), path
        for x, y in zip(a, b):
            _same(x, y, path)
    elif isinstance(a, float) or isinstance(b, float):
        assert math.isclose(a, b, rel_tol=REL, abs_tol=1e-300), (path, a, b)
    else:
        assert a == b, (path, a, b)


def _params(pv):
    from paper_2601_04860_b200 import FusionParams
    return FusionParams(*[float(x) for x in pv[:13]], enable_thin=bool(pv[13]))


def test_thick_thin_checks(gold):
    from dataclasses import asdict

    from paper_2601_04860_b200 import SceneBounds, thick_check, thin_check
    (vg, mask), = _views(gold, "checks")
    bounds = SceneBounds((-4, -4, -4), (4, 4, 4))
    dx = float(gold["checks_dx"])
    for i, line in enumerate(gold["checks"]):
        want = json.loads(str(line))
        p = _params(want["pv"])
        ok, dec = thick_check(np.asarray(want["center"]), dx, want["rho"], vg, mask, p, bounds,
                              voxel_index=(i, 0, 0), view_index=0)
        tdec = thin_check(np.asarray(want["center"]), dx, want["rho"], vg, mask, p,
                          voxel_index=(i, 0, 0))
        assert ok == want["ok"]
        _same(json.loads(json.dumps(asdict(dec))), want["thick"], f"case{i}.thick")
        _same(json.loads(json.dumps(asdict(tdec))), want["thin"], f"case{i}.thin")


def test_thin_check_rod(gold):
    from dataclasses import asdict

    from paper_2601_04860_b200 import FusionParams, thin_check
    (vg, mask), = _views(gold, "rod")
    for line in gold["rod"]:
        want = json.loads(str(line))
        dec = thin_check(np.asarray(want["center"]), want["voxel"], want["rho"], vg, mask,
                         FusionParams())
        _same(json.loads(json.dumps(asdict(dec))), want["thin"])


def test_depth_gradient(gold):
    from paper_2601_04860_b200 import Camera, ViewGeometry, depth_gradient
    cam = Camera(fx=10.0, fy=10.0, cx=4.0, cy=4.0, width=8, height=8, world_from_camera=np.eye(4))
    pix = ((4, 4), (0, 0), (7, 7), (5, 4), (2, 6))
    for i, px in enumerate(pix):
        dexp, n = gold[f"grad{i}_dexp"], gold[f"grad{i}_n"]
        vg = ViewGeometry(cam, None, np.full((8, 8), 1.0, np.float32),
                          np.full((8, 8), 3.0, np.float32), dexp, n, dexp)
        assert depth_gradient(vg, px) == gold["grads"][i]


def test_depth_weight_closed_forms():
    from paper_2601_04860_b200 import depth_weight
    assert depth_weight(2.0, 1.0, 3.0, 4.0) == pytest.approx(1.0)
    assert depth_weight(3.0, 1.0, 3.0, 4.0) == pytest.approx(math.exp(-4.0), rel=1e-12)
    assert depth_weight(2.0, 2.0, 2.0, 4.0, eps=1e-8) == 1.0
    with pytest.raises(ValueError):
        depth_weight(1.0, 3.0, 2.0, 4.0)


def test_fuse_trace_path(gold, tmp_path):
    """fuse(trace_path=...) writes the reference's lines and returns its probabilities."""
    from paper_2601_04860_b200 import (DensityGrid, FusionParams, SceneBounds, VoxelGrid, fuse)
    views = _views(gold, "traced")
    g = int(gold["traced_g"])
    grid = VoxelGrid(g, 1.2, origin=(-1.2, -1.2, -4.2))
    dens = DensityGrid(grid, gold["traced_density"])
    bounds = SceneBounds((-4, -4, -4), (4, 4, 4))
    path = tmp_path / "trace.jsonl"
    og = fuse(grid, dens, views, FusionParams(), bounds=bounds, trace_path=path)
    got = path.read_text().splitlines()
    want = [str(x) for x in gold["traced_lines"]]
    assert len(got) == len(want)
    for a, b in zip(got, want):
        _same(json.loads(a), json.loads(b))
    assert np.allclose(og.probs, gold["traced_probs"], rtol=REL, atol=0)
    kernel = fuse(grid, dens, views, FusionParams(), bounds=bounds)
    assert np.allclose(og.probs, kernel.probs, atol=1e-12)     # test_fusion.py:275
