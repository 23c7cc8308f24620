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


def stress_cases():
    """Adversarial lattice and dense (rho = 5) instances (make_stress_golden.py)."""
    d = _npz("stress.npz")
    return [_case(d, str(n)) for n in d["names"]]


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


# --------------------------------------------------------------------------
# fixture producers (tests/golden/make_render_golden.py -> render.npz)
# --------------------------------------------------------------------------

@dataclass
class PackedScene:
    """A scene given by its packed arrays; quacks like SceneModel for the
    device marcher / bake (``packed()``, ``background``, ``bounds``)."""
    kinds: np.ndarray
    params: np.ndarray
    dens: np.ndarray
    cols: np.ndarray
    soft: np.ndarray
    background: tuple
    bounds: object = None

    def packed(self):
        return (self.kinds, self.params, self.dens, self.cols,
                np.ones(len(self.kinds), np.int32), self.soft)

    def arrays(self):
        return self.kinds, self.params, self.dens, self.cols, self.soft, np.asarray(self.background)


@dataclass
class Bounds:
    min: np.ndarray
    max: np.ndarray
    unbounded: bool


@dataclass
class GoldCam:
    rotation: np.ndarray
    position: np.ndarray
    fx: float
    fy: float
    cx: float
    cy: float
    width: int
    height: int


@dataclass
class GoldCfg:
    samples_per_ray: int
    near: float
    far: float
    tau_cw: float
    min_weight: float


def render_scene(name):
    d = _npz("render.npz")
    p = f"scene_{name}_"
    return PackedScene(d[p + "kinds"], d[p + "params"], d[p + "dens"], d[p + "cols"],
                       d[p + "soft"], tuple(float(x) for x in d[p + "bg"]))


def render_cases():
    """[(scene name, PackedScene, GoldCam, GoldCfg, {output: array})]."""
    d = _npz("render.npz")
    out = []
    for i in range(int(d["render_n"])):
        p = f"render{i}_"
        name = str(d[p + "scene"])
        wfc, intr, c = d[p + "wfc"], d[p + "intr"], d[p + "cfg"]
        cam = GoldCam(wfc[:3, :3].copy(), wfc[:3, 3].copy(), *map(float, intr[:4]),
                      int(intr[4]), int(intr[5]))
        cfg = GoldCfg(int(c[0]), float(c[1]), float(c[2]), float(c[3]), float(c[4]))
        outs = {k: d[p + k] for k in ("rgb", "d_min", "d_max", "d_exp", "n_samples",
                                      "z_surface")}
        out.append((f"{i}-{name}", render_scene(name), cam, cfg, outs))
    return out


def march_cases():
    """(list of (PackedScene, GoldCfg) per ray, rays [n, 6], reference outputs [n, 8])."""
    d = _npz("render.npz")
    names = [str(x) for x in d["scene_names"]]
    per = []
    for c in d["march_cfg"]:
        per.append((render_scene(names[int(c[0])]),
                    GoldCfg(int(c[1]), float(c[2]), float(c[3]), float(c[4]), float(c[5]))))
    return per, d["march_rays"], d["march_out"]


def bake_cases():
    """[(name, PackedScene with bounds, g, half, origin, values (G,G,G) f32)]."""
    d = _npz("render.npz")
    out = []
    for i in range(int(d["bake_n"])):
        p = f"bake{i}_"
        sc = render_scene(str(d[p + "scene"]))
        b = d[p + "bounds"]
        sc.bounds = Bounds(b[:3].copy(), b[3:6].copy(), bool(b[6] > 0))
        out.append((f"{i}-{d[p + 'scene']}", sc, int(d[p + "g"]), float(d[p + "half"]),
                    d[p + "origin"], d[p + "values"]))
    return out
