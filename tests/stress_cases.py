"""Stress inputs for the fusion parity tests (numpy only; no reference import).

Two families (VERDICT round 1 "what's weak" #1):

* ``lattice_case`` -- adversarial geometry on which the kernel's certified
  shortcuts cannot decide: axis-aligned cameras with dyadic intrinsics over a
  dyadic grid, so voxel centres and corners project EXACTLY onto pixel edges
  and onto the frustum borders (u = 0 included, u = 1 excluded), depth maps on
  the same lattice so |x_d - d_exp| equals tau_depth and the thin tau exactly,
  clamped thick segments whose distance equals tau_spatial exactly, masks and
  densities exactly at the gate thresholds, and thin scores exactly at
  thin_accept.  Every fallback of csrc/fuse.cu (exact centre chain, exact
  thick chain, exact corner chain, f64 recount) fires on it.
* ``dense_case`` -- rho = 5 everywhere (every voxel passes the density gate,
  so the early-out never helps) over given view planes with uniform random
  masks, as in the acceptance family (pkg/tests/test_acceptance.py:108).

Both return a dict of packed arrays in the layout of fusion._pack_views
(fusion.py:653-681) plus the grid and the 14-entry parameter vector.
"""

import numpy as np

# FusionParams.as_vector() order (fusion.py:80-87)
PV_NAMES = ("gamma", "beta", "bmax", "lam", "rho_thr", "rho_thin", "thin_pct", "alpha1",
            "thin_accept", "eps", "mask_thr", "thin_floor", "kappa", "enable_thin")


def _pv(**kw):
    base = dict(gamma=1.5, beta=0.5, bmax=16.0, lam=0.0, rho_thr=0.5, rho_thin=2.0,
                thin_pct=0.5, alpha1=4.0, thin_accept=0.625, eps=2.0 ** -30, mask_thr=0.5,
                thin_floor=0.1, kappa=1.0, enable_thin=1.0)
    base.update(kw)
    return np.array([base[k] for k in PV_NAMES], dtype=np.float64)


def _cam(rot, pos, fx, fy, cx, cy, w, h):
    return rot, np.asarray(pos, np.float64), np.array([fx, fy, cx, cy, w, h], np.float64)


# rotations whose columns are the camera axes in world coordinates; the camera
# looks along its -z axis (geometry.py:61-64, fusion.py:170-184)
_ROTS = {
    "-z": np.eye(3),                                              # looks along world -z
    "+z": np.array([[-1.0, 0, 0], [0, 1.0, 0], [0, 0, -1.0]]),     # looks along world +z
    "-x": np.array([[0, 0, 1.0], [0, 1.0, 0], [-1.0, 0, 0]]),      # camera z = world +x
    "-y": np.array([[1.0, 0, 0], [0, 0, 1.0], [0, -1.0, 0]]),      # camera z = world +y
}


def lattice_case(g=32, res=64, seed=0, n_views=8):
    """Adversarial lattice instance (see the module docstring).

    Grid: G voxels over [-1, 1]^3 (dx = 2 / G, dyadic for power-of-two G).
    Views: axis-aligned cameras placed so that one voxel plane (centres, or the
    front / back faces of a plane) lies at depth exactly 2, with fx = fy =
    2 / dx (one pixel per voxel step at depth 2), so lattice offsets project
    to integer or half-integer pixel coordinates.  eps = 2^-30 keeps the
    reference's divisions defined (numba raises on x / 0) while g and the
    thick tolerances stay within the certification margins of the lattice.
    """
    rng = np.random.default_rng(seed)
    dx = 2.0 / g
    half = 0.5 * dx
    centres = -1.0 + (np.arange(g) + 0.5) * dx
    w = h = int(res)
    # fx * (k * dx) / 2 == k * (fx * dx / 2): integral for fx = 2 / dx (one pixel
    # per voxel step at depth 2) -- centres / faces land on pixel edges
    fx = 2.0 / dx
    cams = []
    kinds = ["centre", "front", "back", "border"]
    for v in range(n_views):
        axis = ["-z", "+z", "-x", "-y"][v % 4]
        kind = kinds[(v // 1) % 4]
        rot = _ROTS[axis]
        look = -rot[:, 2]                       # viewing direction in world coordinates
        ax = int(np.argmax(np.abs(look)))
        sgn = np.sign(look[ax])
        # target plane coordinate along the viewing axis (a centre or a face)
        k = int(rng.integers(g // 4, 3 * g // 4))
        plane = centres[k] + {"centre": 0.0, "front": -sgn * half, "back": sgn * half,
                              "border": 0.0}[kind]
        pos = np.zeros(3)
        pos[ax] = plane - sgn * 2.0             # depth of the plane == 2 exactly
        # lateral position on a voxel centre or a face (lattice of dx / 2)
        for a in range(3):
            if a != ax:
                pos[a] = centres[int(rng.integers(g // 4, 3 * g // 4))] + \
                    (half if rng.random() < 0.5 else 0.0)
        # border views: two pixels per voxel step and the principal point off
        # centre, so both frustum borders (u = 0 kept, u = 1 dropped) cut the grid
        f = fx if kind != "border" else 2.0 * fx
        cx = w / 2.0 if kind != "border" else float(w // 4)
        cy = h / 2.0
        cams.append(_cam(rot, pos, f, f, cx, cy, w, h))
    nv = len(cams)
    rots = np.stack([c[0] for c in cams])
    poss = np.stack([c[1] for c in cams])
    intr = np.stack([c[2] for c in cams])
    # depth maps on the lattice: d_exp = 2 + i / 32 * dx * 16 ... multiples of
    # dx / 4 around 2, so |x_d - d_exp| hits tau_depth = 2 dx and the thin tau
    # 3.5 dx exactly for many (voxel, pixel) pairs
    q = dx / 4.0
    dexps = (2.0 + q * rng.integers(-24, 25, size=(nv, h, w))).astype(np.float32)
    span = q * rng.integers(0, 9, size=(nv, h, w))
    dmins = (dexps - span).astype(np.float32)
    dmaxs = (dexps + span).astype(np.float32)
    # clamped thick segments: d_min = x_d + tau_spatial (= dx * g, g = 1 on flat
    # neighbourhoods with lambda = 0) on some pixels, d_max = x_d - dx on others
    sel = rng.random((nv, h, w)) < 0.15
    dmins = np.where(sel, np.float32(2.0 + dx), dmins).astype(np.float32)
    dmaxs = np.where(sel, np.float32(2.0 + 2 * dx), dmaxs).astype(np.float32)
    sel2 = rng.random((nv, h, w)) < 0.15
    dmins = np.where(sel2, np.float32(2.0 - 3 * dx), dmins).astype(np.float32)
    dmaxs = np.where(sel2, np.float32(2.0 - dx), dmaxs).astype(np.float32)
    nsamps = rng.choice(np.array([0, 1, 1, 1, 2, 3], np.int32), size=(nv, h, w))
    # masks exactly at the thresholds (0.1, 0.5, thin_accept 0.625) plus dyadic
    # values in between
    vals = np.array([0.0, 0.1, 0.25, 0.5, 0.5, 0.625, 0.625, 0.75, 0.875, 1.0], np.float32)
    masks = vals[rng.integers(0, len(vals), size=(nv, h, w))]
    # invalid pixels hold zeros in every map (render.py:71-78)
    inv = nsamps == 0
    for a in (dexps, dmins, dmaxs):
        a[inv] = 0.0
    dmins = np.minimum(dmins, dmaxs)
    # density exactly at the gates (rho_thr = 0.5, rho_thin = 2) and above
    dvals = np.array([0.0, 0.5, 2.0, 2.0, 5.0, 5.0], np.float32)
    density = dvals[rng.integers(0, len(dvals), size=g ** 3)].astype(np.float32)
    return dict(g=g, half=1.0, origin=np.array([-1.0, -1.0, -1.0]), dx=dx, density=density,
                rots=rots, poss=poss, intr=intr, masks=masks, dmins=dmins, dmaxs=dmaxs,
                dexps=dexps, nsamps=nsamps.astype(np.int32), pv=_pv(),
                bc=np.zeros(3), bh=np.ones(3), unb=0)


def dense_case(base, g, seed, rho=5.0):
    """rho = 5 everywhere over ``base``'s view planes with uniform random masks
    (refined) and random FusionParams in the acceptance family's ranges
    (test_acceptance.py:108-125).  ``base``: dict / case with packed arrays,
    ``origin`` and ``half`` (the grid keeps the base extent at resolution g)."""
    rng = np.random.default_rng(seed)
    get = (lambda k: base[k]) if isinstance(base, dict) else (lambda k: getattr(base, k))
    masks = rng.random(get("masks").shape, dtype=np.float32)
    pv = _pv(gamma=float(rng.uniform(0.5, 3.0)), beta=float(rng.uniform(0.0, 1.0)),
             bmax=float(rng.uniform(0.0, 20.0)), lam=float(rng.uniform(0.0, 0.3)),
             rho_thr=float(rng.uniform(0.0, 2.0)), rho_thin=float(rng.uniform(0.0, 4.0)),
             thin_pct=float(rng.uniform(0.1, 0.9)), alpha1=float(rng.uniform(0.5, 16.0)),
             thin_accept=float(rng.uniform(0.05, 0.95)), eps=1e-8,
             kappa=float(rng.uniform(0.2, 3.0)))
    half = float(get("half"))
    return dict(g=int(g), half=half, origin=np.asarray(get("origin"), np.float64),
                dx=(2.0 * half) / int(g), density=np.full(int(g) ** 3, rho, np.float32),
                rots=get("rots"), poss=get("poss"), intr=get("intr"), masks=masks,
                dmins=get("dmins"), dmaxs=get("dmaxs"), dexps=get("dexps"),
                nsamps=get("nsamps"), pv=pv, bc=np.asarray(get("bc"), np.float64),
                bh=np.asarray(get("bh"), np.float64), unb=int(get("unb")))
