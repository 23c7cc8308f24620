"""Pin the CPU oracle against the reference's own outputs (golden vectors).

Bit-exact: the oracle restates numba's IEEE evaluation op for op, so every
probability must equal the reference's ``divas.fusion.fuse`` to the last bit
and every refined mask must equal ``divas.segmenter.refine_mask``.
"""

import numpy as np
import pytest

import oracle
from tests import golden_io


def _run(case, early_out=True, nthreads=0):
    return oracle.fuse_packed(case.g, case.origin, case.dx, case.density, case.packed,
                              case.pv, case.bc, case.bh, case.unb,
                              early_out=early_out, nthreads=nthreads)


@pytest.mark.parametrize("case", golden_io.fuzz_cases(), ids=lambda c: c.name)
def test_oracle_matches_reference_fuzz(case):
    r = _run(case)
    assert np.array_equal(r["p"], case.p)


@pytest.mark.parametrize("case", golden_io.stress_cases(), ids=lambda c: c.name)
def test_oracle_matches_reference_stress(case):
    """Adversarial lattice (exact pixel edges, frustum borders, depth-test and
    gate equalities) and dense rho = 5 instances: bit-exact, with and without
    the density early-out."""
    r = _run(case)
    assert np.array_equal(r["p"], case.p)
    r2 = _run(case, early_out=False)
    for k in ("p", "n_thick", "n_thin"):
        assert np.array_equal(r[k], r2[k]), k


@pytest.mark.parametrize("name", ["sop", "small", "g1", "mixed"])
def test_oracle_matches_reference_scenes(name):
    case = golden_io.scene_cases()[name]
    r = _run(case)
    assert np.array_equal(r["p"], case.p)
    # early-out is exact and the result is independent of the thread count
    r2 = _run(case, early_out=False, nthreads=1)
    for k in ("p", "n_thick", "n_thin", "sw", "smw", "st"):
        assert np.array_equal(r[k], r2[k]), k


def test_hand_trace_g1():
    case = golden_io.scene_cases()["g1"]
    r = _run(case)
    assert r["p"][0] == pytest.approx(0.7, abs=1e-6)
    assert r["n_thick"][0] == 1 and r["n_thin"][0] == 0


def test_votes_consistent_with_probability():
    case = golden_io.scene_cases()["sop"]
    r = _run(case)
    denom = r["sw"] + r["n_thin"]
    nz = denom > case.pv[9]
    p = np.zeros_like(r["p"])
    p[nz] = (r["smw"][nz] + r["st"][nz]) / denom[nz]
    assert np.array_equal(p, r["p"])
    assert ((r["n_thick"] + r["n_thin"]) > 0).sum() == (r["p"] != 0).sum() or \
        np.all(r["p"][(r["n_thick"] + r["n_thin"]) == 0] == 0)


@pytest.mark.parametrize("i", range(7))
def test_oracle_refine_matches_reference(i):
    m, z, n, want = golden_io.refine_cases()[i]
    got = oracle.refine(m, z, n)
    assert got.dtype == np.float32
    assert np.array_equal(got, want)


def test_oracle_refine_scene():
    raw, z, refined = golden_io.scene_raw()
    case = golden_io.scene_cases()["sop"]
    for v in range(raw.shape[0]):
        got = oracle.refine(raw[v], z[v], case.nsamps[v])
        assert np.array_equal(got, refined[v])


def test_gradient_padded_semantics():
    """Mixed-resolution sets use the padded (Hmax, Wmax) neighbourhood."""
    case = golden_io.scene_cases()["mixed"]
    g = oracle.gradient_maps(case.dexps, case.dmins, case.dmaxs, case.valids,
                             case.pv[9], case.pv[12])
    assert g.shape == case.masks.shape
    assert np.all((g >= 0) & (g < 1))
    assert np.all(g[case.valids == 0] == 0)
