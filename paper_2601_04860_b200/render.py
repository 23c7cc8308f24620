"""``ViewGeometry`` and the volumetric ray marcher that produces it.

Mirror of /root/reference/pkg/src/divas/render.py.  Maps are (H, W) row-major
``[iy, ix]``; ``valid = n_samples > 0``; invalid pixels hold 0 in every depth
map (render.py:55-78).

The marcher (a fixture producer) runs on the
device: ``render_views_device`` renders any number of same-size cameras in
one ``divas_render`` launch and leaves the planes in HBM, where
``DeviceViews`` / the fusion read them without a host round trip;
``render_view`` / ``march_ray`` keep the reference's host signatures.
Results are bit-identical to the reference's on every pixel the kernel does
not flag ``unsure`` (CUDA's exp vs the C library's; see csrc/render.cu).
"""

from __future__ import annotations

import ctypes
from dataclasses import dataclass

import numpy as np

from . import _native
from ._device import as_device, device, empty, zeros
from .geometry import Camera

__all__ = ["RenderConfig", "ViewGeometry", "RaySample", "march_ray", "march_rays_device",
           "render_view", "render_views_device"]


@dataclass(frozen=True)
class RenderConfig:
    samples_per_ray: int = 192
    near: float = 0.05
    far: float = 8.0
    tau_cw: float = 0.75
    min_weight: float = 1e-4

    def __post_init__(self):                       # render.py:44-50
        if self.samples_per_ray < 1:
            raise ValueError("samples_per_ray must be positive")
        if not self.near < self.far:
            raise ValueError("near must be below far")
        if not 0.0 < self.tau_cw <= 1.0:
            raise ValueError("tau_cw must lie in (0, 1]")


@dataclass
class ViewGeometry:
    camera: Camera
    rgb: np.ndarray        # (H, W, 3) float32 (unused on the hot path)
    d_min: np.ndarray      # (H, W) float32
    d_max: np.ndarray      # (H, W) float32
    d_exp: np.ndarray      # (H, W) float32
    n_samples: np.ndarray  # (H, W) int32
    z_surface: np.ndarray  # (H, W) float32

    @property
    def valid(self) -> np.ndarray:
        return self.n_samples > 0

    def check(self):
        """The D-ordering invariant on every valid pixel (render.py:80-88)."""
        v = self.valid
        assert np.all(self.d_min[v] <= self.d_exp[v] + 1e-6)
        assert np.all(self.d_exp[v] <= self.d_max[v] + 1e-6)
        inv = ~v
        for m in (self.d_min, self.d_max, self.d_exp, self.z_surface):
            assert np.all(m[inv] == 0.0)


@dataclass(frozen=True)
class RaySample:
    rgb: tuple
    d_min: float
    d_max: float
    d_exp: float
    n_samples: int
    z_surface: float

    @property
    def valid(self) -> bool:
        return self.n_samples > 0


def _cfg_struct(cfg) -> _native.RenderCfg:
    return _native.RenderCfg(int(cfg.samples_per_ray), float(cfg.near), float(cfg.far),
                             float(cfg.tau_cw), float(cfg.min_weight))


def render_views_device(scene, cameras, cfg, dev=None, stream=None, unsure=False):
    """Render same-size cameras in one launch; returns a dict of CUDA tensors
    ``rgb`` [nv, H, W, 3], ``d_min``/``d_max``/``d_exp``/``z_surface`` f32 and
    ``n_samples`` i32 [nv, H, W] (+ ``unsure`` u8 [nv, H, W] when asked)."""
    from .fusion import pack_cameras
    from .scene import scene_struct
    cameras = list(cameras)
    if not cameras:
        raise ValueError("no cameras")
    h, w = int(cameras[0].height), int(cameras[0].width)
    if any((int(c.height), int(c.width)) != (h, w) for c in cameras):
        raise ValueError("render_views_device renders cameras of one size per call")
    dev = dev or device()
    st, _keep = scene_struct(scene)
    rc = _cfg_struct(cfg)
    nv = len(cameras)
    cams = as_device(pack_cameras(cameras), np.float64, dev)
    o = dict(rgb=empty((nv, h, w, 3), np.float32, dev), d_min=empty((nv, h, w), np.float32, dev),
             d_max=empty((nv, h, w), np.float32, dev), d_exp=empty((nv, h, w), np.float32, dev),
             n_samples=empty((nv, h, w), np.int32, dev),
             z_surface=empty((nv, h, w), np.float32, dev))
    if unsure:
        o["unsure"] = zeros((nv, h, w), np.uint8, dev)
    P = _native.ptr
    _native.check(_native.lib().divas_render(
        ctypes.byref(st), ctypes.byref(rc), nv, P(cams), h, w, P(o["rgb"]), P(o["d_min"]),
        P(o["d_max"]), P(o["d_exp"]), P(o["n_samples"]), P(o["z_surface"]),
        P(o.get("unsure")), _native.stream_handle(stream)), "render_view")
    o["_cams"] = cams          # keep the camera records alive until the stream runs
    return o


def render_view(scene, camera, cfg) -> ViewGeometry:
    """Render every pixel-center ray of a camera; deterministic."""
    o = render_views_device(scene, [camera], cfg)
    host = {k: v[0].cpu().numpy() for k, v in o.items() if not k.startswith("_")}
    return ViewGeometry(camera, host["rgb"], host["d_min"], host["d_max"], host["d_exp"],
                        host["n_samples"], host["z_surface"])


def march_rays_device(scene, rays, cfg, dev=None, stream=None):
    """``_march`` on unit rays [n, 6] (origin, direction): returns (out [n, 8] f64
    = r, g, b, d_min, d_max, d_exp, n_samples, z_surface; err [n, 4] bounds on
    |out - reference| for r, g, b, d_exp; unsure [n] u8), CUDA tensors."""
    from .scene import scene_struct
    dev = dev or device()
    st, _keep = scene_struct(scene)
    rc = _cfg_struct(cfg)
    r = as_device(rays, np.float64, dev).reshape(-1, 6).contiguous()
    n = r.shape[0]
    out = zeros((n, 8), np.float64, dev)
    err = zeros((n, 4), np.float64, dev)
    uns = zeros((n,), np.uint8, dev)
    P = _native.ptr
    _native.check(_native.lib().divas_march_rays(
        ctypes.byref(st), ctypes.byref(rc), n, P(r), P(out), P(err), P(uns),
        _native.stream_handle(stream)), "march_ray")
    return out, err, uns


def march_ray(scene, ray, cfg) -> RaySample:
    """March a single ray through the scene (render.py:257-267)."""
    o = np.asarray(ray.origin, np.float64).reshape(3)
    d = np.asarray(ray.direction, np.float64).reshape(3)
    out, _err, _u = march_rays_device(scene, np.concatenate([o, d])[None], cfg)
    v = out[0].cpu().numpy()
    return RaySample((float(v[0]), float(v[1]), float(v[2])), float(v[3]), float(v[4]),
                     float(v[5]), int(v[6]), float(v[7]))
