"""Synthetic inputs for the BASELINE.json configurations (bench / tests only).

The reference renders its fixtures with a numba ray marcher and a
region-growing segmenter (out of scope here).  This
module builds inputs of the same shape and statistics directly on the device:

* scene: the ``sphere_on_plane`` profile (/root/reference/pkg/src/divas/
  scenes.py:103-122): hollow sphere (r 0.5, inner 0.45, sigma 46) on a pad
  box (sigma 40, soft edge 0.004) inside a six-wall room;
* cameras: Fibonacci sphere rig (planner.py:64-91), the survey's 5x4
  forward-facing grid (C2) and centroid-zoom views (planner.py:143-160, zoom
  0.47) for C3;
* per-pixel maps: analytic first-hit of the pixel-centre ray, snapped to the
  marcher's midpoint sample lattice (near 0.4, far 12.5, 384 samples): with
  sigma*dt ~ 1.4 the cumulative-weight cutoff 0.75 is reached at the first
  sample inside matter, so d_min = d_max = d_exp = z_surface = that sample
  and n_samples = 1, as the marcher gives on this scene;
* masks: the object-1 silhouette with the segmenter's linear falloff over
  2 px (segmenter.py:115-119);
* density: ``bake_density_grid``'s formula at voxel centres (scene.py:194-201).

Inputs are synthetic, deterministic and bench-only; parity is established on
the golden vectors and on these same inputs against the CPU oracle.
"""

from __future__ import annotations

import math
from dataclasses import dataclass

import numpy as np

CENTER = (0.0, 0.55, 0.0)
SPHERE_R, SPHERE_IN, SPHERE_SIGMA = 0.5, 0.45, 46.0
PAD_C, PAD_H, PAD_SIGMA = (0.0, -0.85, 0.0), (0.3, 0.075, 0.3), 40.0
SOFT = 0.004
ROOM_INNER, ROOM_T = 4.6, 0.2
NEAR, FAR, SPP = 0.4, 12.5, 384
GRID_HALF = 1.2

CONFIGS = {
    "C1": dict(g=128, views="fib", n=8, w=504, h=378),
    "C2": dict(g=256, views="grid5x4", n=20, w=1008, h=756),
    "C3": dict(g=256, views="fib+zoom", n=32, w=1008, h=756),
    "C5": dict(g=512, views="fib", n=128, w=1920, h=1080),
}


def _look_at(pos, tgt):
    pos = np.asarray(pos, np.float64)
    fwd = np.asarray(tgt, np.float64) - pos
    fwd = fwd / np.linalg.norm(fwd)
    up = np.array([0.0, 1.0, 0.0])
    if abs(fwd @ up) > math.cos(math.radians(1.0)):
        up = np.array([1.0, 0.0, 0.0])
    z = -fwd
    x = np.cross(up, z)
    x = x / np.linalg.norm(x)
    y = np.cross(z, x)
    m = np.eye(4)
    m[:3, 0], m[:3, 1], m[:3, 2], m[:3, 3] = x, y, z, pos
    return m


def fibonacci_positions(n, radius=3.3, center=CENTER):
    golden = (1.0 + math.sqrt(5.0)) / 2.0
    i = np.arange(n, dtype=np.float64)
    z = 1.0 - 2.0 * (i + 0.5) / n
    r = np.sqrt(np.maximum(1.0 - z * z, 0.0))
    phi = 2.0 * math.pi * i / golden
    d = np.stack([r * np.cos(phi), z, r * np.sin(phi)], axis=-1)
    return np.asarray(center) + radius * d


@dataclass
class Cam:
    fx: float
    fy: float
    cx: float
    cy: float
    width: int
    height: int
    world_from_camera: np.ndarray

    @property
    def rotation(self):
        return self.world_from_camera[:3, :3]

    @property
    def position(self):
        return self.world_from_camera[:3, 3]


def cameras(kind, n, w, h):
    f = 1.25 * h
    intr = dict(fx=f, fy=f, cx=w / 2.0, cy=h / 2.0, width=w, height=h)
    c = np.asarray(CENTER)
    if kind == "fib":
        return [Cam(world_from_camera=_look_at(p, c), **intr) for p in fibonacci_positions(n)]
    if kind == "grid5x4":
        out = []
        for yy in np.linspace(-0.3, 0.3, 4):
            for xx in np.linspace(-0.4, 0.4, 5):
                out.append(Cam(world_from_camera=_look_at(c + np.array([xx, yy, 3.3]), c), **intr))
        return out[:n]
    if kind == "fib+zoom":
        na = n // 2
        anchors = [Cam(world_from_camera=_look_at(p, c), **intr) for p in fibonacci_positions(na)]
        out = list(anchors)
        # 8 anchors x 2 prompts -> centroid views (zoom 0.47) on the sphere surface
        for a in anchors[:8]:
            x = a.rotation[:, 0]
            for s in (-0.22, 0.22):
                d = (c + s * x) - a.position
                d = d / np.linalg.norm(d)
                # first hit of the prompt ray on the outer sphere
                oc = a.position - c
                b = oc @ d
                t = -b - math.sqrt(max(b * b - (oc @ oc - SPHERE_R ** 2), 0.0))
                tgt = a.position + t * d
                pos = a.position + (1.0 - 0.47) * (tgt - a.position)
                out.append(Cam(world_from_camera=_look_at(pos, tgt), **intr))
        return out[:n]
    raise ValueError(kind)


def _boxes():
    cx, cy, cz = CENTER
    t, inner = ROOM_T, ROOM_INNER
    d = inner + t
    walls = [((cx - d, cy, cz), (t, inner + 2 * t, inner + 2 * t)),
             ((cx + d, cy, cz), (t, inner + 2 * t, inner + 2 * t)),
             ((cx, cy - d, cz), (inner + 2 * t, t, inner + 2 * t)),
             ((cx, cy + d, cz), (inner + 2 * t, t, inner + 2 * t)),
             ((cx, cy, cz - d), (inner + 2 * t, inner + 2 * t, t)),
             ((cx, cy, cz + d), (inner + 2 * t, inner + 2 * t, t))]
    return [(PAD_C, PAD_H)] + walls


def render_maps(cam, device="cpu"):
    """(d_min, d_max, d_exp, n_samples, z_surface, object-1 hit) for one camera."""
    import torch
    h, w = cam.height, cam.width
    dt = (FAR - NEAR) / SPP
    iy, ix = torch.meshgrid(torch.arange(h, device=device, dtype=torch.float64),
                            torch.arange(w, device=device, dtype=torch.float64), indexing="ij")
    xc = (ix + 0.5 - cam.cx) / cam.fx
    yc = (cam.cy - (iy + 0.5)) / cam.fy
    R = torch.tensor(cam.rotation, dtype=torch.float64, device=device)
    # elementwise IEEE ops only (no matmul / norm kernels, whose FMA use and
    # reduction order differ between devices): the same bits on the CPU and
    # the GPU, so the reference arm (CPU) sees this arm's exact masks
    d = torch.stack([R[0, 0] * xc + R[0, 1] * yc - R[0, 2], R[1, 0] * xc + R[1, 1] * yc - R[1, 2],
                     R[2, 0] * xc + R[2, 1] * yc - R[2, 2]], dim=-1)
    nrm = torch.sqrt(d[..., 0] * d[..., 0] + d[..., 1] * d[..., 1] + d[..., 2] * d[..., 2])
    d = d / nrm.unsqueeze(-1)
    o = torch.tensor(cam.position, dtype=torch.float64, device=device)
    inf = torch.full((h, w), float("inf"), dtype=torch.float64, device=device)
    # sphere (outer surface entry; hollow interior only matters past the cutoff)
    oc = [float(cam.position[j]) - CENTER[j] for j in range(3)]
    b = d[..., 0] * oc[0] + d[..., 1] * oc[1] + d[..., 2] * oc[2]
    disc = b * b - ((oc[0] * oc[0] + oc[1] * oc[1] + oc[2] * oc[2]) - SPHERE_R ** 2)
    t_s = torch.where(disc >= 0, -b - torch.sqrt(disc.clamp(min=0)), inf)
    t_s = torch.where(t_s > NEAR, t_s, inf)
    t_best, obj = t_s, torch.where(torch.isfinite(t_s), 1, 0)
    for k, (bc, bh) in enumerate(_boxes()):
        bc = torch.tensor(bc, dtype=torch.float64, device=device)
        bh = torch.tensor(bh, dtype=torch.float64, device=device) + SOFT * 0.5
        inv = 1.0 / torch.where(d.abs() < 1e-12, torch.full_like(d, 1e-12), d)
        ta = (bc - bh - o) * inv
        tb = (bc + bh - o) * inv
        tmin = torch.minimum(ta, tb).amax(-1)
        tmax = torch.maximum(ta, tb).amin(-1)
        t_b = torch.where((tmax >= tmin) & (tmax > NEAR), tmin.clamp(min=NEAR), inf)
        closer = t_b < t_best
        t_best = torch.where(closer, t_b, t_best)
        obj = torch.where(closer, 2 + k, obj)
    hit = torch.isfinite(t_best) & (t_best < FAR)
    k = torch.ceil((t_best - NEAR) / dt - 0.5).clamp(min=0)
    t_k = NEAR + (k + 0.5) * dt
    zero = torch.zeros((h, w), dtype=torch.float32, device=device)
    dmap = torch.where(hit, t_k, 0.0).to(torch.float32)
    n = hit.to(torch.int32)
    return dmap, dmap.clone(), dmap.clone(), n, dmap.clone(), (obj == 1) & hit, zero


def silhouette_mask(core):
    """Segmenter confidence: 1 on the core, 1 - dist/2 within 2 px (EDT falloff)."""
    import torch
    conf = core.to(torch.float32)
    h, w = core.shape
    c = core
    for dy in range(-1, 2):
        for dx in range(-1, 2):
            r = math.hypot(dx, dy)
            if r == 0 or r >= 2:
                continue
            sh = torch.zeros_like(c)
            ys, ye = max(dy, 0), h + min(dy, 0)
            xs, xe = max(dx, 0), w + min(dx, 0)
            sh[ys:ye, xs:xe] = c[ys - dy:ye - dy, xs - dx:xe - dx]
            conf = torch.maximum(conf, sh.to(torch.float32) * (1.0 - r / 2.0))
    return conf


def density_grid(g, device="cpu"):
    """bake_density_grid of the scene at voxel centres: (G,G,G) f32 [ix,iy,iz].

    Primitives whose soft-edged box cannot reach the grid (the room walls)
    contribute exactly 0 and are skipped.
    """
    import torch
    dx = 2.0 * GRID_HALF / g
    origin = np.asarray(CENTER) - GRID_HALF
    ax = [origin[a] + (torch.arange(g, device=device, dtype=torch.float64) + 0.5) * dx
          for a in range(3)]
    lo, hi = origin, origin + 2 * GRID_HALF
    boxes = [(bc, bh) for bc, bh in _boxes()
             if all(bc[j] - bh[j] - SOFT <= hi[j] and bc[j] + bh[j] + SOFT >= lo[j] for j in range(3))]
    out = torch.empty((g, g, g), dtype=torch.float32, device=device)
    Y, Z = torch.meshgrid(ax[1], ax[2], indexing="ij")
    step = max(1, (1 << 22) // (g * g))
    for i0 in range(0, g, step):
        X = ax[0][i0:i0 + step].view(-1, 1, 1)
        dist = torch.sqrt((X - CENTER[0]) ** 2 + (Y - CENTER[1]) ** 2 + (Z - CENTER[2]) ** 2)
        sd = torch.maximum(dist - SPHERE_R, SPHERE_IN - dist)
        val = torch.where(sd <= 0, SPHERE_SIGMA, 0.0)
        for bc, bh in boxes:
            qx = ((X - bc[0]).abs() - bh[0]).expand_as(dist)
            qy = ((Y - bc[1]).abs() - bh[1]).expand_as(dist)
            qz = ((Z - bc[2]).abs() - bh[2]).expand_as(dist)
            outside = torch.sqrt(qx.clamp(min=0) ** 2 + qy.clamp(min=0) ** 2 + qz.clamp(min=0) ** 2)
            inside = torch.maximum(torch.maximum(qx, qy), qz).clamp(max=0)
            fall = (1.0 - (outside + inside) / SOFT).clamp(0.0, 1.0)
            val = torch.maximum(val, PAD_SIGMA * fall)
        out[i0:i0 + step] = val.to(torch.float32)
    return out, origin, dx


_ROOM_COLORS = ((0.30, 0.30, 0.34), (0.32, 0.30, 0.30), (0.26, 0.28, 0.26),
                (0.34, 0.34, 0.38), (0.28, 0.31, 0.36), (0.33, 0.29, 0.33))


def scene_model():
    """The ``sphere_on_plane`` SceneModel (scenes.py:103-122 with _room,
    scenes.py:77-100) as the package's mirror types, for the device marcher
    and bake."""
    from paper_2601_04860_b200.geometry import SceneBounds
    from paper_2601_04860_b200.scene import SceneModel, ScenePrimitive
    sphere = ScenePrimitive("sphere", {"center": CENTER, "radius": SPHERE_R,
                                       "inner_radius": SPHERE_IN},
                            density=SPHERE_SIGMA, color=(0.85, 0.2, 0.15), object_id=1)
    pad = ScenePrimitive("box", {"center": PAD_C, "half_extents": PAD_H}, density=PAD_SIGMA,
                         color=(0.1, 0.14, 0.2), object_id=2, soft_edge=SOFT)
    walls = tuple(ScenePrimitive("box", {"center": bc, "half_extents": bh}, density=40.0,
                                 color=col, object_id=90 + i, soft_edge=SOFT)
                  for i, ((bc, bh), col) in enumerate(zip(_boxes()[1:], _ROOM_COLORS)))
    return SceneModel((sphere, pad) + walls, SceneBounds((-4.9, -4.4, -4.9), (4.9, 5.5, 4.9)),
                      background=(0.02, 0.02, 0.04))


@dataclass
class Workload:
    name: str
    g: int
    origin: np.ndarray
    dx: float
    density: object        # (G^3,) f32 tensor
    cams: list
    raw_masks: object      # [nv, h, w] f32 tensor (unrefined)
    z_surface: object
    dmins: object
    dmaxs: object
    dexps: object
    nsamps: object

    @property
    def nv(self):
        return len(self.cams)

    @property
    def shape(self):
        return tuple(self.raw_masks.shape)

    def updates(self):
        return self.g ** 3 * self.nv


def make(name, device="cpu", g=None, n_views=None, width=None, height=None, source="analytic"):
    """Inputs of a BASELINE config.  ``source="marcher"`` takes d_min / d_max /
    d_exp / n_samples / z_surface from the reference's ray marcher and the
    density from its bake, both run on the device and bit-identical to the
    reference's (render.cu); the masks stay the analytic silhouette."""
    import torch
    cfg = dict(CONFIGS[name])
    if g:
        cfg["g"] = g
    if n_views:
        cfg["n"] = n_views
    if width:
        cfg["w"] = width
    if height:
        cfg["h"] = height
    cams = cameras(cfg["views"], cfg["n"], cfg["w"], cfg["h"])
    planes = {k: [] for k in ("raw", "z", "dmin", "dmax", "dexp", "n")}
    for cam in cams:
        dmin, dmax, dexp, n, z, core, _ = render_maps(cam, device)
        planes["raw"].append(silhouette_mask(core))
        planes["z"].append(z)
        planes["dmin"].append(dmin)
        planes["dmax"].append(dmax)
        planes["dexp"].append(dexp)
        planes["n"].append(n)
    st = {k: torch.stack(v).contiguous() for k, v in planes.items()}
    dens, origin, dx = density_grid(cfg["g"], device)
    if source == "marcher":
        from paper_2601_04860_b200.geometry import VoxelGrid
        from paper_2601_04860_b200.render import RenderConfig, render_views_device
        from paper_2601_04860_b200.scene import bake_density_device
        sc = scene_model()
        o = render_views_device(sc, cams, RenderConfig(samples_per_ray=SPP, near=NEAR, far=FAR),
                                dev=torch.device(device), unsure=True)
        if int(o["unsure"].sum()):
            raise RuntimeError("marcher flagged pixels whose bits are not certified")
        st.update(z=o["z_surface"], dmin=o["d_min"], dmax=o["d_max"], dexp=o["d_exp"],
                  n=o["n_samples"])
        dens = bake_density_device(sc, VoxelGrid(cfg["g"], GRID_HALF, origin),
                                   dev=torch.device(device))
    elif source != "analytic":
        raise ValueError(source)
    return Workload(name, cfg["g"], origin, dx, dens.reshape(-1).contiguous(), cams, st["raw"],
                    st["z"], st["dmin"], st["dmax"], st["dexp"], st["n"])
