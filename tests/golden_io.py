"""Loaders for the committed golden vectors (tests/golden/*.npz).

The vectors were produced by the reference itself (tests/golden/make_golden.py);
nothing here reads /root/reference at run time.
"""

import os
from dataclasses import dataclass

import numpy as np

GOLDEN = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")
_cache = {}


def _npz(name):
    if name not in _cache:
        _cache[name] = dict(np.load(os.path.join(GOLDEN, name)))
    return _cache[name]


@dataclass
class FuseCase:
    name: str
    g: int
    origin: np.ndarray
    dx: float
    half: float
    density: np.ndarray
    rots: np.ndarray
    poss: np.ndarray
    intr: np.ndarray
    masks: np.ndarray
    dmins: np.ndarray
    dmaxs: np.ndarray
    dexps: np.ndarray
    nsamps: np.ndarray
    pv: np.ndarray
    bc: np.ndarray
    bh: np.ndarray
    unb: int
    p: np.ndarray          # expected probabilities, flat G^3 (reference fuse)

    @property
    def valids(self):
        return (self.nsamps > 0).astype(np.uint8)

    @property
    def packed(self):
        return (self.rots, self.poss, self.intr, self.masks, self.dmins, self.dmaxs,
                self.dexps, self.nsamps, self.valids)


def _case(d, prefix):
    g = int(d[f"{prefix}_g"])
    p = np.zeros(g ** 3, dtype=np.float64)
    p[d[f"{prefix}_p_idx"]] = d[f"{prefix}_p_val"]
    return FuseCase(
        name=prefix, g=g, origin=d[f"{prefix}_origin"], dx=float(d[f"{prefix}_dx"]), half=float(d[f"{prefix}_half"]),
        density=d[f"{prefix}_density"], rots=d[f"{prefix}_rots"], poss=d[f"{prefix}_poss"],
        intr=d[f"{prefix}_intr"], masks=d[f"{prefix}_masks"], dmins=d[f"{prefix}_dmins"],
        dmaxs=d[f"{prefix}_dmaxs"], dexps=d[f"{prefix}_dexps"], nsamps=d[f"{prefix}_nsamps"],
        pv=d[f"{prefix}_pv"], bc=d[f"{prefix}_bc"], bh=d[f"{prefix}_bh"],
        unb=int(d[f"{prefix}_unb"]), p=p)


def fuzz_cases(limit=None):
    d = _npz("fuzz.npz")
    n = int(d["n_trials"])
    if limit is not None:
        n = min(n, limit)
    return [_case(d, f"t{t:03d}") for t in range(n)]


def scene_cases():
    d = _npz("scene.npz")
    return {k: _case(d, k) for k in ("sop", "small", "g1", "mixed")}


def scene_raw():
    d = _npz("scene.npz")
    return d["sop_raw_masks"], d["sop_z"], d["sop_refined"]


def refine_cases():
    d = _npz("refine.npz")
    return [(d[f"c{i}_mask"], d[f"c{i}_z"], d[f"c{i}_n"], d[f"c{i}_out"])
            for i in range(int(d["n_cases"]))]
