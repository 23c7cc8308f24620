"""Pin the fixture producers' CPU oracle against the reference (render.npz).

``oracle/divas_oracle_render.c`` restates ``render._march`` / ``_render``
(numba) and ``bake_density_grid`` (numpy) op for op, with the C library's
exp -- the same one numba's math.exp calls -- so every output must equal
the reference's bit for bit.  Also: the host-side mirrors (RenderConfig /
ScenePrimitive validation, SceneModel.packed) against the reference's.
"""

import numpy as np
import pytest

import oracle
from tests import golden_io


def _bits(a):
    a = np.asarray(a)
    return a.view(np.uint32) if a.dtype == np.float32 else a


@pytest.mark.parametrize("case", golden_io.render_cases(), ids=lambda c: c[0])
def test_oracle_render_matches_reference(case):
    _name, sc, cam, cfg, ref = case
    o = oracle.render(sc.arrays(), cam, cfg)
    for k, v in ref.items():
        assert np.array_equal(_bits(o[k]), _bits(v)), k


def test_oracle_march_matches_reference():
    per, rays, ref = golden_io.march_cases()
    for i, (sc, cfg) in enumerate(per):
        o = oracle.march(sc.arrays(), cfg, rays[i])[0]
        assert np.array_equal(o, ref[i]), i


@pytest.mark.parametrize("case", golden_io.bake_cases(), ids=lambda c: c[0])
def test_oracle_bake_matches_reference(case):
    _name, sc, g, half, origin, ref = case
    v = oracle.bake(sc.arrays(), g, half, origin, sc.bounds)
    assert np.array_equal(_bits(v), _bits(ref))


def test_render_config_validation():
    from paper_2601_04860_b200.render import RenderConfig
    RenderConfig()
    for bad in (dict(samples_per_ray=0), dict(near=2.0, far=1.0), dict(tau_cw=0.0),
                dict(tau_cw=1.5)):
        with pytest.raises(ValueError):
            RenderConfig(**bad)


def test_scene_mirror_packs_like_reference():
    """SceneModel.packed() of the mirror == the reference's packed arrays
    (the ``mixed`` scene of make_render_golden.py)."""
    from paper_2601_04860_b200.geometry import SceneBounds
    from paper_2601_04860_b200.scene import SceneModel, ScenePrimitive
    bounds = SceneBounds((-5, -5, -5), (5, 5, 5))
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
    ref = golden_io.render_scene("mixed")
    k, p, d, c, _o, s = mixed.packed()
    assert np.array_equal(k, ref.kinds) and np.array_equal(p, ref.params)
    assert np.array_equal(d, ref.dens) and np.array_equal(c, ref.cols)
    assert np.array_equal(s, ref.soft) and mixed.background == ref.background


def test_scene_primitive_validation():
    from paper_2601_04860_b200.scene import ScenePrimitive
    ok = dict(params={"center": (0, 0, 0), "radius": 1.0}, density=1.0, color=(1, 1, 1),
              object_id=1)
    ScenePrimitive("sphere", **ok)
    with pytest.raises(ValueError):
        ScenePrimitive("cone", **ok)
    with pytest.raises(ValueError):
        ScenePrimitive("sphere", **{**ok, "density": -1.0})
    with pytest.raises(ValueError):
        ScenePrimitive("sphere", **{**ok, "object_id": 0})
    with pytest.raises(ValueError):
        ScenePrimitive("sphere", **{**ok, "params": {"center": (0, 0, 0), "radius": 1.0,
                                                     "inner_radius": 1.0}})
    with pytest.raises(ValueError):
        ScenePrimitive("box", **{**ok, "params": {"center": (0, 0, 0),
                                                  "half_extents": (1, 0, 1)}})


def test_bench_scene_is_reference_sphere_on_plane():
    """workloads.scene_model() (the bench's scene) packs exactly like the
    reference's get_profile("sphere_on_plane").scene."""
    import workloads
    ref = golden_io.render_scene("sop")
    k, p, d, c, _o, s = workloads.scene_model().packed()
    assert np.array_equal(k, ref.kinds) and np.array_equal(p, ref.params)
    assert np.array_equal(d, ref.dens) and np.array_equal(c, ref.cols)
    assert np.array_equal(s, ref.soft)
    assert workloads.scene_model().background == ref.background
