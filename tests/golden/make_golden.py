"""Generate the golden vectors that pin the oracle -- run HERE, not on the GPU box.

Imports the reference package (``/root/reference/pkg``) from a writable copy
(numba ``cache=True`` writes next to its sources) and records inputs plus the
reference's own outputs:

* ``fuzz.npz``    -- acceptance criterion #1's random family
  (``pkg/tests/test_acceptance.py:66-145``, seed 20260811): packed inputs
  exactly as ``fusion._pack_views`` builds them and ``divas.fusion.fuse``'s
  probabilities (stored sparse).  200 trials.
* ``refine.npz``  -- ``divas.segmenter.refine_mask`` on rendered views
  (``pkg/tests/test_segmenter.py`` fixtures) with constant, random and
  partially invalidated inputs, plus constant-depth and all-invalid cases.
* ``scene.npz``   -- the ``sphere_on_plane`` profile end to end at a reduced
  size (G=64, 8 Fibonacci views at 126x94): ``render_view`` ->
  ``segment_from_prompt`` -> ``refine_mask`` -> ``bake_density_grid`` ->
  ``fuse``; plus the ``small_instance`` of ``pkg/tests/test_fusion.py:82-96``,
  the G=1 hand trace (``test_fusion.py:303-316``) and a mixed-resolution view
  set (padded-gradient semantics, SURVEY.md section 7 hard part 3).

Usage:  python tests/golden/make_golden.py [--ref /root/reference/pkg]
"""

from __future__ import annotations

import argparse
import importlib.util
import os
import shutil
import sys

import numpy as np

OUT = os.path.dirname(os.path.abspath(__file__))


def _import_reference(ref_pkg):
    work = "/tmp/divas_golden_ref"
    if not os.path.isdir(work):
        shutil.copytree(ref_pkg, work)
    os.environ.setdefault("NUMBA_CACHE_DIR", "/tmp/divas_golden_nbcache")
    sys.path.insert(0, os.path.join(work, "src"))
    import divas  # noqa: F401
    spec = importlib.util.spec_from_file_location(
        "ref_acceptance", os.path.join(work, "tests", "test_acceptance.py"))
    ta = importlib.util.module_from_spec(spec)
    spec.loader.exec_module(ta)
    return ta


def _pack(views):
    from divas.fusion import _pack_views
    return _pack_views(views)


def _sparse(p):
    flat = p.reshape(-1)
    idx = np.flatnonzero(flat).astype(np.int32)
    return idx, flat[idx]


def _record(store, prefix, grid, dens, views, params, bounds, probs):
    from divas.fusion import _bounds_arrays
    rots, poss, intr, masks, dmins, dmaxs, dexps, nsamps, valids = _pack(views)
    bc, bh, unb = _bounds_arrays(bounds)
    idx, val = _sparse(probs)
    store.update({
        f"{prefix}_g": np.int64(grid.resolution),
        f"{prefix}_origin": np.asarray(grid.origin, dtype=np.float64),
        f"{prefix}_dx": np.float64(grid.voxel_size()),
        f"{prefix}_half": np.float64(grid.half_extents[0]),
        f"{prefix}_density": np.asarray(dens.values, dtype=np.float32),
        f"{prefix}_rots": rots, f"{prefix}_poss": poss, f"{prefix}_intr": intr,
        f"{prefix}_masks": masks, f"{prefix}_dmins": dmins, f"{prefix}_dmaxs": dmaxs,
        f"{prefix}_dexps": dexps, f"{prefix}_nsamps": nsamps,
        f"{prefix}_pv": params.as_vector(),
        f"{prefix}_bc": np.asarray(bc, dtype=np.float64),
        f"{prefix}_bh": np.asarray(bh, dtype=np.float64),
        f"{prefix}_unb": np.int64(unb),
        f"{prefix}_p_idx": idx, f"{prefix}_p_val": val,
    })
    assert np.array_equal(valids, (nsamps > 0).astype(np.uint8))


def make_fuzz(ta, n_trials=200):
    from divas.fusion import fuse
    rng = np.random.default_rng(20260811)
    store = {}
    for t in range(n_trials):
        scene, grid, dens, views, params = ta._random_instance(rng)
        probs = fuse(grid, dens, views, params, bounds=scene.bounds, workers=2).probs
        _record(store, f"t{t:03d}", grid, dens, views, params, scene.bounds, probs)
    store["n_trials"] = np.int64(n_trials)
    np.savez_compressed(os.path.join(OUT, "fuzz.npz"), **store)


def make_refine():
    from divas.geometry import Camera, SceneBounds
    from divas.render import RenderConfig, render_view
    from divas.scene import SceneModel, ScenePrimitive
    from divas.segmenter import ConfidenceMask, refine_mask
    bounds = SceneBounds((-8, -8, -8), (8, 8, 8))
    intr = dict(fx=120.0, fy=120.0, cx=48.0, cy=48.0, width=96, height=96)
    cfg = RenderConfig(samples_per_ray=256, near=0.5, far=8.0)
    cam = Camera(world_from_camera=np.eye(4), **intr)
    sphere = ScenePrimitive("sphere", {"center": (0, 0, -2.0), "radius": 0.7},
                            density=400.0, color=(0.9, 0.2, 0.1), object_id=1)
    wall = ScenePrimitive("box", {"center": (0, 0, -5.0), "half_extents": (7, 7, 0.5)},
                          density=400.0, color=(0.2, 0.4, 0.9), object_id=2)
    vg = render_view(SceneModel((sphere, wall), bounds), cam, cfg)
    rng = np.random.default_rng(7)
    cases = []
    z, n = vg.z_surface, vg.n_samples
    cases.append((np.full(z.shape, 0.8, np.float32), z, n))
    cases.append((rng.random(z.shape).astype(np.float32), z, n))
    n2 = n.copy()
    n2[:10, :10] = 0
    cases.append((np.ones(z.shape, np.float32), z, n2))
    cases.append((rng.random(z.shape).astype(np.float32), np.full_like(z, 2.5), n))
    cases.append((rng.random((5, 7)).astype(np.float32), rng.random((5, 7)).astype(np.float32),
                  np.zeros((5, 7), np.int32)))
    zr = (rng.random((37, 53)) * 9.0).astype(np.float32)
    nr = (rng.random((37, 53)) < 0.7).astype(np.int32) * 5
    cases.append((rng.random((37, 53)).astype(np.float32), zr, nr))
    # extreme dynamic range + negative depths + exact-boundary mask values
    ze = rng.normal(0, 1e3, (16, 16)).astype(np.float32)
    me = rng.choice(np.array([0.0, 0.1, 0.5, 1.0, 0.3333333], np.float32), (16, 16))
    cases.append((me, ze, np.ones((16, 16), np.int32)))
    store = {"n_cases": np.int64(len(cases))}
    for i, (m, zz, nn) in enumerate(cases):
        from divas.render import ViewGeometry
        h, w = zz.shape
        cam_i = Camera(fx=10.0, fy=10.0, cx=w / 2, cy=h / 2, width=w, height=h,
                       world_from_camera=np.eye(4))
        zeros = np.zeros((h, w), np.float32)
        v = ViewGeometry(cam_i, np.zeros((h, w, 3), np.float32), zeros, zeros, zeros,
                         nn.astype(np.int32), zz.astype(np.float32))
        out = refine_mask(ConfidenceMask(m), v).values
        store[f"c{i}_mask"] = m
        store[f"c{i}_z"] = zz.astype(np.float32)
        store[f"c{i}_n"] = nn.astype(np.int32)
        store[f"c{i}_out"] = out
    np.savez_compressed(os.path.join(OUT, "refine.npz"), **store)


def make_scene():
    from divas.fusion import FusionParams, fuse
    from divas.geometry import Camera, SceneBounds, VoxelGrid, look_at
    from divas.planner import fibonacci_sample
    from divas.render import RenderConfig, ViewGeometry, render_view
    from divas.scene import DensityGrid, SceneModel, ScenePrimitive, bake_density_grid
    from divas.scenes import get_profile
    from divas.segmenter import ConfidenceMask, refine_mask, segment_from_prompt
    store = {}
    # sphere_on_plane, reduced C1 (G=64, 8 views @126x94)
    prof = get_profile("sphere_on_plane")
    W, H = 126, 94
    intr = dict(fx=1.25 * H, fy=1.25 * H, cx=W / 2.0, cy=H / 2.0, width=W, height=H)
    cams = fibonacci_sample(8, prof.rig_radius, prof.rig_center, intr)
    views, raw = [], []
    for cam in cams:
        vg = render_view(prof.scene, cam, prof.render)
        m = segment_from_prompt(vg, (W // 2, H // 2), prof.segmenter) if vg.valid[H // 2, W // 2] \
            else ConfidenceMask(np.zeros((H, W), np.float32))
        rm = refine_mask(m, vg)
        raw.append((m.values, vg.z_surface, vg.n_samples, rm.values))
        views.append((vg, rm))
    grid = prof.make_grid(64)
    dens = bake_density_grid(prof.scene, grid)
    probs = fuse(grid, dens, views, prof.fusion, bounds=prof.scene.bounds).probs
    _record(store, "sop", grid, dens, views, prof.fusion, prof.scene.bounds, probs)
    import io as _io
    from divas.io import write_fmap, write_vgrid
    from divas.fusion import OccupancyGrid as _OG
    buf = _io.BytesIO()
    write_vgrid(buf, _OG(grid, probs), unbounded=prof.scene.bounds.unbounded)
    store["sop_vgrid_bytes"] = np.frombuffer(buf.getvalue(), dtype=np.uint8)
    buf = _io.BytesIO()
    write_fmap(buf, views[0][0].d_exp)
    store["sop_fmap_bytes"] = np.frombuffer(buf.getvalue(), dtype=np.uint8)
    store["sop_raw_masks"] = np.stack([r[0] for r in raw])
    store["sop_z"] = np.stack([r[1] for r in raw])
    store["sop_refined"] = np.stack([r[3] for r in raw])
    # project_grid_overlay of the fused grid onto every view (fusion.py:846-865)
    from divas.fusion import OccupancyGrid, project_grid_overlay
    og = OccupancyGrid(grid, probs)
    store["sop_overlay"] = np.stack([project_grid_overlay(og, vg, bounds=prof.scene.bounds)
                                     for vg, _m in views]).astype(np.uint8)
    store["sop_overlay_thr03"] = np.stack([project_grid_overlay(og, vg, threshold=0.3)
                                           for vg, _m in views]).astype(np.uint8)
    # small_instance (test_fusion.py:82-96), sigma=2.5, g=14
    bounds = SceneBounds((-4, -4, -4), (4, 4, 4))
    INTR = dict(fx=96.0, fy=96.0, cx=32.0, cy=32.0, width=64, height=64)
    CFG = RenderConfig(samples_per_ray=192, near=0.5, far=7.0)
    sphere = ScenePrimitive("sphere", {"center": (0, 0, -3.0), "radius": 0.8},
                            density=2.5, color=(0.8, 0.2, 0.2), object_id=1)
    scene = SceneModel((sphere,), bounds)
    cams = [Camera(world_from_camera=np.eye(4), **INTR),
            Camera(world_from_camera=look_at((3.0, 0.3, -3.0), (0, 0, -3.0)), **INTR)]
    sviews = []
    for c in cams:
        vg = render_view(scene, c, CFG)
        sviews.append((vg, ConfidenceMask(np.where(vg.valid, 0.9, 0.0).astype(np.float32),
                                          refined=True)))
    g14 = VoxelGrid(14, 1.2, origin=(-1.2, -1.2, -4.2))
    d14 = bake_density_grid(scene, g14)
    p = FusionParams()
    _record(store, "small", g14, d14, sviews, p, bounds,
            fuse(g14, d14, sviews, p, bounds=bounds).probs)
    # G=1 hand trace (test_fusion.py:303-316): expected p = 0.7
    cam = Camera(fx=10.0, fy=10.0, cx=4.0, cy=4.0, width=8, height=8, world_from_camera=np.eye(4))
    mk = lambda v: np.full((8, 8), v, dtype=np.float32)  # noqa: E731
    vg1 = ViewGeometry(cam, np.zeros((8, 8, 3), np.float32), mk(1.5), mk(2.5), mk(2.0),
                       np.full((8, 8), 30, np.int32), mk(2.0))
    m1 = ConfidenceMask(mk(0.7), refined=True)
    g1 = VoxelGrid(1, 0.05, origin=(-0.05, -0.05, -2.05))
    d1 = DensityGrid(g1, np.full((1, 1, 1), 5.0, np.float32))
    _record(store, "g1", g1, d1, [(vg1, m1)], p, None, fuse(g1, d1, [(vg1, m1)], p).probs)
    # mixed resolution: two views of the small scene at different sizes, and an
    # unbounded variant -- exercises padded gradient maps and contraction
    intr2 = dict(fx=60.0, fy=60.0, cx=20.0, cy=15.0, width=40, height=30)
    c3 = Camera(world_from_camera=look_at((0.4, 2.8, -2.6), (0, 0, -3.0)), **intr2)
    vg3 = render_view(scene, c3, CFG)
    mixed = sviews + [(vg3, ConfidenceMask(np.where(vg3.valid, 0.8, 0.05).astype(np.float32),
                                           refined=True))]
    unb = SceneBounds((-1, -1, -4), (1, 1, -2), unbounded=True)
    pm = fuse(g14, d14, mixed, p, bounds=unb).probs
    _record(store, "mixed", g14, d14, mixed, p, unb, pm)
    og14 = OccupancyGrid(g14, pm)
    store["mixed_overlay"] = np.stack([project_grid_overlay(og14, vg, threshold=0.2, bounds=unb)
                                       .astype(np.uint8).ravel() for vg, _m in mixed[:2]])
    np.savez_compressed(os.path.join(OUT, "scene.npz"), **store)


def _store_views(store, prefix, views):
    store[f"{prefix}_nv"] = np.int64(len(views))
    for i, (vg, m) in enumerate(views):
        c = vg.camera
        store[f"{prefix}_v{i}_intr"] = np.array([c.fx, c.fy, c.cx, c.cy, c.width, c.height],
                                                dtype=np.float64)
        store[f"{prefix}_v{i}_w2c"] = np.asarray(c.world_from_camera, dtype=np.float64)
        for k in ("d_min", "d_max", "d_exp", "n_samples", "z_surface"):
            store[f"{prefix}_v{i}_{k}"] = np.asarray(getattr(vg, k))
        store[f"{prefix}_v{i}_mask"] = np.asarray(m.values, dtype=np.float32)


def make_trace():
    """thick_check / thin_check / depth_gradient / fuse(trace_path) of the
    reference (test_fusion.py fixtures)."""
    import json
    import tempfile
    from dataclasses import asdict
    from divas.fusion import (FusionParams, depth_gradient, fuse, thick_check, thin_check)
    from divas.geometry import Camera, SceneBounds, VoxelGrid, look_at
    from divas.render import RenderConfig, ViewGeometry, render_view
    from divas.scene import SceneModel, ScenePrimitive, bake_density_grid
    from divas.segmenter import ConfidenceMask
    bounds = SceneBounds((-4, -4, -4), (4, 4, 4))
    INTR = dict(fx=96.0, fy=96.0, cx=32.0, cy=32.0, width=64, height=64)
    CFG = RenderConfig(samples_per_ray=192, near=0.5, far=7.0)
    store = {}

    def small(sigma, g):
        sphere = ScenePrimitive("sphere", {"center": (0, 0, -3.0), "radius": 0.8},
                                density=sigma, color=(0.8, 0.2, 0.2), object_id=1)
        scene = SceneModel((sphere,), bounds)
        cams = [Camera(world_from_camera=np.eye(4), **INTR),
                Camera(world_from_camera=look_at((3.0, 0.3, -3.0), (0, 0, -3.0)), **INTR)]
        views = []
        for c in cams:
            vg = render_view(scene, c, CFG)
            views.append((vg, ConfidenceMask(np.where(vg.valid, 0.9, 0.0).astype(np.float32),
                                             refined=True)))
        grid = VoxelGrid(g, 1.2, origin=(-1.2, -1.2, -4.2))
        return scene, grid, bake_density_grid(scene, grid), views

    # traced fuse (test_fusion.py:269-278)
    scene, grid, dens, views = small(2.5, 8)
    p = FusionParams()
    with tempfile.TemporaryDirectory() as td:
        path = os.path.join(td, "t.jsonl")
        og = fuse(grid, dens, views, p, bounds=scene.bounds, trace_path=path)
        store["traced_lines"] = np.array(open(path).read().splitlines())
    store["traced_probs"] = og.probs
    store["traced_g"] = np.int64(8)
    store["traced_density"] = np.asarray(dens.values, np.float32)
    _store_views(store, "traced", views)
    # thick_check cases (test_fusion.py:99-142) on small_instance(300, 16) view 0
    scene, grid, dens, views = small(300.0, 16)
    vg, mask = views[0]
    dx = grid.voxel_size()
    tau = (p.base_tolerance_multiplier + p.max_bonus) * dx
    cases = [((0.0, 0.0, -2.2 - dx / 2), 300.0, p), ((0.0, 0.0, -2.2 - 10 * tau), 300.0, p),
             ((0, 0, -2.25), 0.1, p), ((0, 0, -3.0), 2.0, FusionParams(per_sample_bonus=100.0,
                                                                       max_bonus=3.0)),
             ((0.05, -0.02, -2.21), 300.0, FusionParams(depth_range_factor=0.3)),
             ((0.0, 0.0, 5.0), 300.0, p)]
    recs = []
    for i, (c, rho, pp) in enumerate(cases):
        ok, dec = thick_check(np.asarray(c, float), dx, rho, vg, mask, pp, scene.bounds,
                              voxel_index=(i, 0, 0), view_index=0)
        tdec = thin_check(np.asarray(c, float), dx, rho, vg, mask, pp, voxel_index=(i, 0, 0))
        recs.append(json.dumps({"ok": ok, "thick": asdict(dec), "thin": asdict(tdec),
                                "center": list(map(float, c)), "rho": rho,
                                "pv": pp.as_vector().tolist()}))
    store["checks"] = np.array(recs)
    store["checks_dx"] = np.float64(dx)
    _store_views(store, "checks", [(vg, mask)])
    # thin_check on the rod (test_fusion.py:145-167)
    rod = ScenePrimitive("capsule", {"p0": (0, -1, -3.0), "p1": (0, 1, -3.0), "radius": 0.02},
                         density=8.0, color=(0.9, 0.3, 0.1), object_id=1)
    rvg = render_view(SceneModel((rod,), bounds), Camera(world_from_camera=np.eye(4), **INTR), CFG)
    rmask = ConfidenceMask(np.where(rvg.valid, 0.95, 0.0).astype(np.float32), refined=True)
    rrecs = []
    for c, vox, rho in (((0, 0, -3.0), 0.04, 8.0), ((0.01, 0.3, -3.0), 0.04, 8.0),
                        ((0, 0, -3.0), 0.04, 0.5), ((0.0, 0.0, -2.0), 0.2, 8.0)):
        tdec = thin_check(np.asarray(c, float), vox, rho, rvg, rmask, p)
        rrecs.append(json.dumps({"thin": asdict(tdec), "center": list(map(float, c)),
                                 "voxel": vox, "rho": rho}))
    store["rod"] = np.array(rrecs)
    _store_views(store, "rod", [(rvg, rmask)])
    # depth_gradient (test_fusion.py:34-58) on hand-built views
    grads = []
    for i, pix in enumerate(((4, 4), (0, 0), (7, 7), (5, 4), (2, 6))):
        cam = Camera(fx=10.0, fy=10.0, cx=4.0, cy=4.0, width=8, height=8,
                     world_from_camera=np.eye(4))
        rng = np.random.default_rng(i)
        dexp = (2.0 + rng.random((8, 8))).astype(np.float32)
        dexp[:, 5:] = 200.0 if i == 0 else dexp[:, 5:]
        n = np.full((8, 8), 20, np.int32)
        n[0, 0] = 0
        gv = ViewGeometry(cam, np.zeros((8, 8, 3), np.float32), np.full((8, 8), 1.0, np.float32),
                          np.full((8, 8), 3.0, np.float32), dexp, n, dexp)
        grads.append(depth_gradient(gv, pix))
        store[f"grad{i}_dexp"] = dexp
        store[f"grad{i}_n"] = n
    store["grads"] = np.array(grads)
    np.savez_compressed(os.path.join(OUT, "trace.npz"), **store)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--ref", default="/root/reference/pkg")
    ap.add_argument("--only", default="fuzz,refine,scene,trace")
    args = ap.parse_args()
    ta = _import_reference(args.ref)
    todo = args.only.split(",")
    if "refine" in todo:
        make_refine()
    if "scene" in todo:
        make_scene()
    if "trace" in todo:
        make_trace()
    if "fuzz" in todo:
        make_fuzz(ta)


if __name__ == "__main__":
    main()
