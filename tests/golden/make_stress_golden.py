"""Generate the stress golden vectors -- run HERE (needs the reference), not on the GPU box.

Imports the reference package from a writable copy (as make_golden.py does)
and records, for inputs built by ``tests/stress_cases.py``, the reference's
own ``divas.fusion.fuse`` probabilities:

* ``lattice*`` -- adversarial lattice instances (exact pixel edges, frustum
  borders, depth-test equalities, gate thresholds): where the kernel's
  certified shortcuts must hand over to the exact chains;
* ``dense*``   -- rho = 5 everywhere (no density early-out) with uniform random
  masks and random FusionParams, over view planes of acceptance criterion #1's
  random family (``pkg/tests/test_acceptance.py:66-127``, a separate seed) and
  over the golden ``sphere_on_plane`` views.

Output: ``tests/golden/stress.npz`` (same per-case keys as fuzz.npz).

Usage:  python tests/golden/make_stress_golden.py [--ref /root/reference/pkg]
"""

from __future__ import annotations

import argparse
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.dirname(os.path.dirname(HERE)))

from tests import stress_cases  # noqa: E402
from tests.golden.make_golden import _import_reference, _record  # noqa: E402

SEED_DENSE = 20261019


def _reference_objects(c):
    """(VoxelGrid, DensityGrid, [(ViewGeometry, ConfidenceMask)], FusionParams, bounds)."""
    from divas.fusion import FusionParams
    from divas.geometry import Camera, SceneBounds, VoxelGrid
    from divas.render import ViewGeometry
    from divas.scene import DensityGrid
    from divas.segmenter import ConfidenceMask
    g = int(c["g"])
    grid = VoxelGrid(g, float(c["half"]), origin=np.asarray(c["origin"], np.float64))
    assert grid.voxel_size() == float(c["dx"]), (grid.voxel_size(), c["dx"])
    dens = DensityGrid(grid, np.asarray(c["density"], np.float32).reshape(g, g, g))
    views = []
    for i in range(c["rots"].shape[0]):
        fx, fy, cx, cy, w, h = c["intr"][i]
        w, h = int(w), int(h)
        m4 = np.eye(4)
        m4[:3, :3] = c["rots"][i]
        m4[:3, 3] = c["poss"][i]
        cam = Camera(fx=fx, fy=fy, cx=cx, cy=cy, width=w, height=h, world_from_camera=m4)
        sl = np.s_[i, :h, :w]
        vg = ViewGeometry(cam, np.zeros((h, w, 3), np.float32), c["dmins"][sl].copy(),
                          c["dmaxs"][sl].copy(), c["dexps"][sl].copy(), c["nsamps"][sl].copy(),
                          c["dexps"][sl].copy())
        views.append((vg, ConfidenceMask(np.asarray(c["masks"][sl], np.float32).copy(),
                                         refined=True)))
    pv = np.asarray(c["pv"], np.float64)
    params = FusionParams(*[float(x) for x in pv[:13]], enable_thin=bool(pv[13]))
    bounds = None
    if int(c["unb"]):
        bounds = SceneBounds(tuple(c["bc"] - c["bh"]), tuple(c["bc"] + c["bh"]), unbounded=True)
    return grid, dens, views, params, bounds


def _fuzz_views(ta, rng):
    """View planes + grid of one acceptance-#1 instance (dict of packed arrays)."""
    from divas.fusion import _bounds_arrays, _pack_views
    scene, grid, dens, views, params = ta._random_instance(rng)
    rots, poss, intr, masks, dmins, dmaxs, dexps, nsamps, _valids = _pack_views(views)
    bc, bh, unb = _bounds_arrays(scene.bounds)
    return dict(rots=rots, poss=poss, intr=intr, masks=masks, dmins=dmins, dmaxs=dmaxs,
                dexps=dexps, nsamps=nsamps, origin=np.asarray(grid.origin, np.float64),
                half=float(grid.half_extents[0]), bc=np.asarray(bc, np.float64),
                bh=np.asarray(bh, np.float64), unb=int(unb))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--ref", default="/root/reference/pkg")
    args = ap.parse_args()
    ta = _import_reference(args.ref)
    from divas.fusion import fuse
    from tests import golden_io
    store = {}
    names = []

    def record(name, c):
        grid, dens, views, params, bounds = _reference_objects(c)
        og = fuse(grid, dens, views, params, bounds=bounds, workers=8)
        _record(store, name, grid, dens, views, params, bounds, og.probs)
        names.append(name)
        nz = int((og.probs != 0).sum())
        print(f"{name}: G={grid.resolution} views={len(views)} nonzero p={nz} "
              f"occupied={int((og.probs >= 0.5).sum())}", flush=True)

    for i, (g, res) in enumerate([(32, 64), (32, 48), (16, 40), (64, 64)]):
        record(f"lattice{i}", stress_cases.lattice_case(g=g, res=res, seed=100 + i))
    rng = np.random.default_rng(SEED_DENSE)
    for i in range(6):
        base = _fuzz_views(ta, rng)
        g = int(rng.integers(24, 41))
        record(f"dense{i}", stress_cases.dense_case(base, g, seed=SEED_DENSE + i))
    sop = golden_io.scene_cases()["sop"]
    record("dense_sop", stress_cases.dense_case(sop, 48, seed=SEED_DENSE + 99))
    store["names"] = np.array(names)
    np.savez_compressed(os.path.join(HERE, "stress.npz"), **store)
    print("wrote", os.path.join(HERE, "stress.npz"),
          os.path.getsize(os.path.join(HERE, "stress.npz")) // 1024, "KiB")


if __name__ == "__main__":
    main()
