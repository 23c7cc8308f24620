"""Stress parity on the GPU: the adversarial lattice (exact pixel edges, frustum
borders, depth-test / gate / thin-accept equalities), the dense rho = 5 family
(no density early-out) and larger instances of both, against the reference's
golden probabilities and the CPU oracle (votes, sums, p bit-exact).

The lattice is built so the kernel's certified shortcuts cannot decide; the
fallback counters (``divas_fuse_args.fallbacks``) must show that each exact
chain ran -- centre projection (fusion.py:170-192), thick pair (:257-303),
corner chain (:315-341) and the f64 support recount (:361-367) -- and the
result must still equal the oracle's bit for bit.
"""

import numpy as np
import pytest

import oracle
from tests import golden_io, stress_cases
from tests.gpu_cases import device_views, grid_ns

pytestmark = pytest.mark.gpu

KEYS = ("n_thick", "n_thin", "sw", "smw", "st")


def _case_obj(name, c):
    """A golden_io.FuseCase-like object from a stress_cases dict."""
    p = np.zeros(int(c["g"]) ** 3)
    return golden_io.FuseCase(name=name, g=int(c["g"]), origin=np.asarray(c["origin"]),
                              dx=float(c["dx"]), half=float(c["half"]), density=c["density"],
                              rots=c["rots"], poss=c["poss"], intr=c["intr"], masks=c["masks"],
                              dmins=c["dmins"], dmaxs=c["dmaxs"], dexps=c["dexps"],
                              nsamps=c["nsamps"], pv=c["pv"], bc=np.asarray(c["bc"]),
                              bh=np.asarray(c["bh"]), unb=int(c["unb"]), p=p)


def _gpu(case, fb=None):
    import torch
    from paper_2601_04860_b200 import _native
    from paper_2601_04860_b200.fusion import Fuser
    from tests.gpu_cases import bounds_ns
    dev = torch.device("cuda", 0)
    dv = device_views(case, dev)
    dens = torch.from_numpy(np.ascontiguousarray(case.density, np.float32).reshape(-1)).to(dev)
    fuser = Fuser(grid_ns(case), case.pv, bounds_ns(case))
    if fb is None:
        fb = torch.zeros(_native.NFALLBACK, dtype=torch.int64, device=dev)
    out = fuser.run(dens, dv, stats=True, occ=True, fallbacks=fb)
    torch.cuda.synchronize()
    return {k: v.cpu().numpy() for k, v in out.items() if k != "workspace"}, fb


def _oracle(case):
    return oracle.fuse_packed(case.g, case.origin, case.dx, case.density, case.packed, case.pv,
                              case.bc, case.bh, case.unb, early_out=False)


def _assert_same(got, ref, case):
    for k in KEYS:
        assert np.array_equal(got[k], ref[k]), (case.name, k)
    assert np.array_equal(got["probs"], ref["p"]), case.name
    assert np.array_equal(got["occ"].astype(bool), ref["p"] >= 0.5), case.name


@pytest.mark.parametrize("case", golden_io.stress_cases(), ids=lambda c: c.name)
def test_stress_goldens_bit_exact(case):
    got, _fb = _gpu(case)
    assert np.array_equal(got["probs"], case.p), case.name     # the reference's fuse
    _assert_same(got, _oracle(case), case)


def test_lattice_fires_every_exact_fallback():
    import torch
    from paper_2601_04860_b200 import _native
    fb = torch.zeros(_native.NFALLBACK, dtype=torch.int64, device="cuda")
    for case in golden_io.stress_cases():
        if case.name.startswith("lattice"):
            got, _ = _gpu(case, fb)
            _assert_same(got, _oracle(case), case)
    counts = dict(zip(_native.FALLBACKS, fb.cpu().tolist()))
    for site in ("centre", "thick", "corners", "recount"):
        assert counts[site] > 0, counts


def test_thin_sum_paths_both_run_and_agree():
    """fuse_reduce's thin sum: the view-order sum, certified exact in every
    order, for the default parameters (every thin vote's t is an f32 mask
    value); the reference's value sort where the certificate fails (random
    thin_percent_cover > thin_accept: t = support / npix votes).  Both
    bit-identical to the oracle."""
    import torch
    from paper_2601_04860_b200 import _native
    sop = golden_io.scene_cases()["sop"]
    # defaults: no sort at all
    got, fb = _gpu(sop)
    assert np.array_equal(got["probs"], sop.p)
    counts = dict(zip(_native.FALLBACKS, fb.cpu().tolist()))
    assert counts["thin_sort"] == 0, counts
    # random parameters with thin_percent_cover > thin_accept: sorted sums
    sorted_hits = 0
    for seed in range(6):
        c = stress_cases.dense_case(sop, 48, seed=900 + seed)
        c["pv"][6], c["pv"][8] = 0.9, 0.3           # thin_pct, thin_accept
        case = _case_obj(f"dense_sort{seed}", c)
        fb = torch.zeros(_native.NFALLBACK, dtype=torch.int64, device="cuda")
        got, fb = _gpu(case, fb)
        _assert_same(got, _oracle(case), case)
        sorted_hits += int(fb[_native.FALLBACKS.index("thin_sort")].item())
    assert sorted_hits > 0


@pytest.mark.parametrize("seed", [0, 1])
def test_lattice_larger_vs_oracle(seed):
    """Bigger lattices (G = 64, 128 x 128 px) than the committed goldens."""
    c = stress_cases.lattice_case(g=64, res=128, seed=500 + seed, n_views=12)
    case = _case_obj(f"lattice_big{seed}", c)
    got, fb = _gpu(case)
    _assert_same(got, _oracle(case), case)
    assert int(fb.sum().item()) > 0


@pytest.mark.parametrize("g", [64, 128])
def test_dense_sop_views_vs_oracle(g):
    """rho = 5 everywhere over the sphere_on_plane golden views (8 x 126 x 94),
    uniform random masks, random FusionParams: every (voxel, view) pair goes
    through the projections (Fuzz row)."""
    sop = golden_io.scene_cases()["sop"]
    case = _case_obj(f"dense_sop{g}", stress_cases.dense_case(sop, g, seed=7 + g))
    got, _fb = _gpu(case)
    _assert_same(got, _oracle(case), case)
    assert int(got["n_thin"].sum() + got["n_thick"].sum()) > 0
