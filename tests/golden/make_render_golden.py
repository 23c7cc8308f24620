"""Golden vectors for the fixture producers -- run HERE.

Imports the reference package from a writable copy (as ``make_golden.py``
does) and records, for a set of scenes, the reference's own outputs of

* ``render_view`` (``/root/reference/pkg/src/divas/render.py:270-292``):
  rgb, d_min, d_max, d_exp, n_samples, z_surface per pixel;
* ``march_ray`` (``render.py:257-267``) on explicit rays;
* ``bake_density_grid`` (``scene.py:194-201``), bounded and unbounded
  (spherical contraction, ``geometry.py:242-256``).

Scenes: the ``pkg/tests/test_render.py`` fixtures (sphere at several
densities, opaque wall, empty, near-transparent), the ``sphere_on_plane``
profile (sphere shell + soft pad + six-wall room, 384 samples per ray) seen
from Fibonacci cameras, and a mixed scene with a capsule, soft edges and a
hollow sphere.  Output: ``render.npz`` next to this file.

Usage:  python tests/golden/make_render_golden.py [--ref /root/reference/pkg]
"""

from __future__ import annotations

import argparse
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


def _scenes():
    from divas.geometry import SceneBounds
    from divas.scene import SceneModel, ScenePrimitive
    from divas.scenes import get_profile
    bounds = SceneBounds((-5, -5, -5), (5, 5, 5))

    def sphere(sigma):
        return SceneModel((ScenePrimitive("sphere", {"center": (0, 0, -3.0), "radius": 0.8},
                                          density=sigma, color=(0.9, 0.1, 0.1), object_id=1),),
                          bounds)

    wall = SceneModel((ScenePrimitive("box", {"center": (0, 0, -2.5),
                                              "half_extents": (4.0, 4.0, 0.5)},
                                      density=500.0, color=(0.2, 0.8, 0.2), object_id=1),),
                      bounds)
    mixed = SceneModel((
        ScenePrimitive("capsule", {"p0": (-0.6, -0.3, -2.6), "p1": (0.7, 0.4, -3.4),
                                   "radius": 0.18}, density=30.0, color=(0.2, 0.7, 0.3),
                       object_id=1, soft_edge=0.05),
        ScenePrimitive("sphere", {"center": (0.3, -0.2, -3.2), "radius": 0.6,
                                  "inner_radius": 0.5}, density=12.0, color=(0.8, 0.3, 0.1),
                       object_id=2, soft_edge=0.02),
        ScenePrimitive("box", {"center": (0.0, 0.0, -4.5), "half_extents": (2.0, 2.0, 0.2)},
                       density=8.0, color=(0.3, 0.3, 0.35), object_id=3, soft_edge=0.1),
    ), bounds, background=(0.05, 0.02, 0.1))
    transparent = SceneModel((ScenePrimitive("sphere", {"center": (0, 0, -3.0), "radius": 0.8},
                                             density=1e-9, color=(1, 1, 1), object_id=1),),
                             bounds)
    prof = get_profile("sphere_on_plane")
    return dict(sphere4=sphere(4.0), sphere50=sphere(50.0), sphere1_5=sphere(1.5),
                wall=wall, empty=SceneModel((), bounds), mixed=mixed,
                transparent=transparent, sop=prof.scene), prof


def _pack_scene(prefix, scene, d):
    kinds, params, dens, cols, _oids, soft = scene.packed()
    d[prefix + "kinds"] = kinds
    d[prefix + "params"] = params
    d[prefix + "dens"] = dens
    d[prefix + "cols"] = cols
    d[prefix + "soft"] = soft
    d[prefix + "bg"] = np.asarray(scene.background, np.float64)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--ref", default="/root/reference/pkg")
    a = ap.parse_args()
    _import_reference(a.ref)
    from divas.geometry import Camera, Ray, SceneBounds, VoxelGrid, look_at
    from divas.planner import fibonacci_sample
    from divas.render import RenderConfig, march_ray, render_view
    from divas.scene import SceneModel, bake_density_grid

    scenes, prof = _scenes()
    d = {}
    for name, sc in scenes.items():
        _pack_scene(f"scene_{name}_", sc, d)
    d["scene_names"] = np.array(list(scenes))

    def front(res, f=1.6):
        return Camera(fx=f * res, fy=f * res, cx=res / 2, cy=res / 2, width=res, height=res,
                      world_from_camera=np.eye(4))

    cfg = RenderConfig(samples_per_ray=256, near=0.5, far=6.0, tau_cw=0.75)
    sop_intr = dict(fx=1.25 * 96, fy=1.25 * 96, cx=48.0, cy=36.0, width=96, height=72)
    sop_cams = fibonacci_sample(4, 3.3, prof.rig_center, sop_intr)
    mixed_cam = Camera(fx=70.0, fy=66.0, cx=23.5, cy=19.0, width=48, height=40,
                       world_from_camera=look_at((0.4, 0.5, 0.2), (0.0, 0.0, -3.2)))
    cases = [
        ("sphere4", front(64), cfg),
        ("sphere50", front(64), cfg),
        ("sphere1_5", front(64), RenderConfig(samples_per_ray=128, near=0.5, far=6.0, tau_cw=0.3)),
        ("sphere1_5", front(64), RenderConfig(samples_per_ray=128, near=0.5, far=6.0, tau_cw=0.9)),
        ("wall", front(16), RenderConfig(samples_per_ray=128, near=0.5, far=6.0)),
        ("wall", front(16), RenderConfig(samples_per_ray=256, near=0.5, far=6.0, tau_cw=1.0)),
        ("empty", front(64), cfg),
        ("transparent", front(32), cfg),
        ("mixed", mixed_cam, RenderConfig(samples_per_ray=200, near=0.3, far=7.0, tau_cw=0.8,
                                          min_weight=1e-3)),
    ] + [("sop", c, prof.render) for c in sop_cams]
    d["render_n"] = np.int64(len(cases))
    for i, (name, cam, rc) in enumerate(cases):
        vg = render_view(scenes[name], cam, rc)
        p = f"render{i}_"
        d[p + "scene"] = np.array(name)
        d[p + "wfc"] = cam.world_from_camera
        d[p + "intr"] = np.array([cam.fx, cam.fy, cam.cx, cam.cy, cam.width, cam.height],
                                 np.float64)
        d[p + "cfg"] = np.array([rc.samples_per_ray, rc.near, rc.far, rc.tau_cw, rc.min_weight],
                                np.float64)
        for k in ("rgb", "d_min", "d_max", "d_exp", "n_samples", "z_surface"):
            d[p + k] = getattr(vg, k)

    # march_ray on explicit rays (unit directions from Ray's normalisation)
    rng = np.random.default_rng(20261018)
    rays, outs, rscene = [], [], []
    for name, n in (("sop", 24), ("mixed", 24), ("sphere4", 8)):
        sc = scenes[name]
        rc = prof.render if name == "sop" else cfg
        for _ in range(n):
            if name == "sop":
                o = np.asarray(prof.rig_center) + rng.normal(size=3) * 1.5
                tgt = np.asarray(prof.rig_center) + rng.normal(size=3) * 0.4
            else:
                o = rng.normal(size=3) * 0.3
                tgt = np.array([0.0, 0.0, -3.0]) + rng.normal(size=3) * 0.7
            ray = Ray(o, tgt - o)
            s = march_ray(sc, ray, rc)
            rays.append(np.concatenate([ray.origin, ray.direction]))
            outs.append([*s.rgb, s.d_min, s.d_max, s.d_exp, float(s.n_samples), s.z_surface])
            rscene.append([list(scenes).index(name),
                           rc.samples_per_ray, rc.near, rc.far, rc.tau_cw, rc.min_weight])
    d["march_rays"] = np.asarray(rays)
    d["march_out"] = np.asarray(outs)
    d["march_cfg"] = np.asarray(rscene, np.float64)

    # bake_density_grid
    bakes = [
        ("sop", VoxelGrid(32, 1.2, np.asarray(prof.rig_center) - 1.2), None),
        ("mixed", VoxelGrid(24, 1.0, np.array([-1.0, -1.0, -4.0])), None),
        ("mixed", VoxelGrid(20, 6.0, np.array([-6.0, -6.0, -9.0])),
         SceneBounds((-1.5, -1.2, -4.6), (1.5, 1.2, -1.4), unbounded=True)),
    ]
    d["bake_n"] = np.int64(len(bakes))
    for i, (name, grid, bnd) in enumerate(bakes):
        sc = scenes[name]
        if bnd is not None:
            sc = SceneModel(sc.primitives, bnd, sc.background)
        dg = bake_density_grid(sc, grid)
        p = f"bake{i}_"
        d[p + "scene"] = np.array(name)
        d[p + "g"] = np.int64(grid.resolution)
        d[p + "half"] = np.float64(grid.half_extent)
        d[p + "origin"] = grid.origin
        d[p + "bounds"] = np.concatenate([sc.bounds.min, sc.bounds.max,
                                          [1.0 if sc.bounds.unbounded else 0.0]])
        d[p + "values"] = dg.values
    np.savez_compressed(os.path.join(OUT, "render.npz"), **d)
    print("wrote render.npz:", len(cases), "renders,", len(rays), "rays,", len(bakes), "bakes")


if __name__ == "__main__":
    main()
