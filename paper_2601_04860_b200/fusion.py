"""Multi-view voxel fusion on the B200 (stages (b) and (c) of the path).

Drop-in for the reference's fusion entry points
(/root/reference/pkg/src/divas/fusion.py):

* ``FusionParams`` (:46-106) and ``OccupancyGrid`` (:109-123) -- same fields,
  validation, ``as_vector`` layout and JSON helpers;
* ``fuse(grid, density, views, params, bounds=None, workers=None,
  trace_path=None)`` (:692-724) -- same signature, same ValueErrors, same
  probabilities (integer votes and occupancy bit-exact; p equal to the last
  bit except where CUDA's ``exp`` and glibc's differ by an ulp in a thick
  weight);
* ``project_grid_overlay`` (:846-865);
* threshold / extract (``probs >= thr`` and ``np.argwhere``, ablation.py:109).

Extensions, not in the reference: ``fuse_with_stats`` (votes and sorted
sums), ``DeviceViews`` / ``Fuser`` for device-resident repeated fusion and
slab sharding (``vox_range``), and ``threshold_device`` / ``extract_device``.

All arithmetic runs in libdivas_b200.so (csrc/*.cu); this module validates,
packs and moves data.  There is no CPU fallback.
"""

from __future__ import annotations

import ctypes
import json
from dataclasses import asdict, dataclass, replace

import numpy as np

from . import _native
from ._device import as_device, device, empty
from .trace import (ThickPathDecision, ThinPathDecision, depth_gradient, depth_weight,
                    thick_check, thin_check)

__all__ = [
    "FusionParams", "OccupancyGrid", "FusionStats", "DeviceViews", "Fuser",
    "fuse", "fuse_with_stats", "refine_and_fuse", "project_grid_overlay",
    "threshold", "extract", "threshold_device", "extract_device", "gradient_maps_device",
    "pack_cameras", "bounds_arrays",
    "ThickPathDecision", "ThinPathDecision", "depth_gradient", "depth_weight", "thick_check",
    "thin_check",
]


# ---------------------------------------------------------------------------
# parameter / result types
# ---------------------------------------------------------------------------

@dataclass(frozen=True)
class FusionParams:
    """Kernel hyperparameters (fusion.py:46-106; the code defaults are authoritative)."""

    base_tolerance_multiplier: float = 1.5   # gamma
    per_sample_bonus: float = 0.5            # beta
    max_bonus: float = 16.0
    depth_range_factor: float = 0.1          # lambda_range
    density_thresh: float = 0.5
    thin_density_thresh: float = 2.0
    thin_percent_cover: float = 0.5
    depth_falloff: float = 4.0               # alpha1
    thin_accept: float = 0.6
    eps: float = 1e-8
    mask_threshold: float = 0.5
    thin_mask_floor: float = 0.1
    grad_kappa: float = 1.0
    enable_thin: bool = True

    def __post_init__(self):
        for name in ("base_tolerance_multiplier", "per_sample_bonus", "max_bonus",
                     "depth_range_factor", "density_thresh", "thin_density_thresh",
                     "thin_percent_cover", "depth_falloff", "eps"):
            if getattr(self, name) < 0:
                raise ValueError(f"{name} must be >= 0")
        if not 0.0 < self.thin_accept < 1.0:
            raise ValueError("thin acceptance threshold must lie in (0, 1)")
        if self.mask_threshold != 0.5:
            raise ValueError("mask threshold is fixed at 0.5")

    def as_vector(self) -> np.ndarray:
        return np.array([
            self.base_tolerance_multiplier, self.per_sample_bonus, self.max_bonus,
            self.depth_range_factor, self.density_thresh, self.thin_density_thresh,
            self.thin_percent_cover, self.depth_falloff, self.thin_accept,
            self.eps, self.mask_threshold, self.thin_mask_floor, self.grad_kappa,
            1.0 if self.enable_thin else 0.0,
        ], dtype=np.float64)

    def to_dict(self) -> dict:
        return asdict(self)

    @classmethod
    def from_dict(cls, d: dict) -> "FusionParams":
        return cls(**d)

    def save(self, path):
        with open(path, "w") as f:
            json.dump(self.to_dict(), f, indent=2)

    @classmethod
    def load(cls, path) -> "FusionParams":
        with open(path) as f:
            return cls.from_dict(json.load(f))

    def with_overrides(self, **kw) -> "FusionParams":
        return replace(self, **kw)


@dataclass
class OccupancyGrid:
    """Fused probabilities on a VoxelGrid layout, (G, G, G) float64 [ix, iy, iz]."""

    grid: object
    probs: np.ndarray
    version: int = 0

    def __post_init__(self):
        g = self.grid.resolution
        self.probs = np.asarray(self.probs, dtype=np.float64).reshape(g, g, g)

    def check(self):
        assert np.all(np.isfinite(self.probs))
        assert self.probs.min() >= 0.0 and self.probs.max() <= 1.0


@dataclass
class FusionStats:
    """Per-voxel integer votes and value-sorted sums.

    p == (smw + st) / (sw + n_thin) where that denominator exceeds eps, else 0.
    """

    n_thick: np.ndarray   # (G,G,G) int32 -- views whose thick path passed
    n_thin: np.ndarray    # (G,G,G) int32 -- accepted thin scores
    sw: np.ndarray        # (G,G,G) f64   -- sum of thick depth weights
    smw: np.ndarray       # (G,G,G) f64   -- sum of m * w
    st: np.ndarray        # (G,G,G) f64   -- sum of accepted thin scores
    gated: int            # voxels that passed the exact density gate


def _params_vector(params) -> np.ndarray:
    if hasattr(params, "as_vector"):
        return np.asarray(params.as_vector(), dtype=np.float64)
    pv = np.asarray(params, dtype=np.float64)
    if pv.shape != (_native.NPARAM,):
        raise ValueError("params vector must have 14 entries")
    return pv


def bounds_arrays(bounds):
    """(centre, half, unbounded) as the kernel takes them (fusion.py:542-546)."""
    if bounds is None or not bounds.unbounded:
        return np.zeros(3), np.ones(3), 0
    return (np.asarray(bounds.center, dtype=np.float64).reshape(3),
            np.asarray(bounds.half, dtype=np.float64).reshape(3), 1)


def _check_layout(grid, density):
    """fusion.py:701-704."""
    if density.grid.resolution != grid.resolution or \
            not np.allclose(density.grid.origin, grid.origin) or \
            density.grid.half_extents != grid.half_extents:
        raise ValueError("density grid layout does not match the fusion grid")


# ---------------------------------------------------------------------------
# device-resident view set
# ---------------------------------------------------------------------------

def pack_cameras(cameras) -> np.ndarray:
    """[nv, 18] f64 records: rotation (row-major), position, fx fy cx cy w h."""
    out = np.zeros((len(cameras), _native.CAM_STRIDE), dtype=np.float64)
    for i, c in enumerate(cameras):
        out[i, 0:9] = np.asarray(c.rotation, dtype=np.float64).reshape(9)
        out[i, 9:12] = np.asarray(c.position, dtype=np.float64).reshape(3)
        out[i, 12:18] = (c.fx, c.fy, c.cx, c.cy, float(c.width), float(c.height))
    return out


class DeviceViews:
    """A view set resident in HBM as padded SoA planes ``[nv, hm, wm]``.

    Layout as ``fusion._pack_views`` builds it (fusion.py:653-681): the largest
    view sets (hm, wm); smaller views occupy the top-left corner; padding is
    zero (so it is invalid: ``n_samples == 0``).  ``masks`` holds the refined
    confidences the fusion consumes; ``z_surface`` (optional) lets
    ``refine()`` produce them on device from ``raw_masks``.
    """

    def __init__(self, cams, masks, dmins, dmaxs, dexps, nsamps, z_surface=None,
                 raw_masks=None, sizes=None):
        self.cams = cams
        self.masks = masks
        self.dmins = dmins
        self.dmaxs = dmaxs
        self.dexps = dexps
        self.nsamps = nsamps
        self.z_surface = z_surface
        self.raw_masks = raw_masks
        self.sizes = sizes

    @property
    def nv(self):
        return int(self.masks.shape[0])

    @property
    def hm(self):
        return int(self.masks.shape[1])

    @property
    def wm(self):
        return int(self.masks.shape[2])

    @property
    def device(self):
        return self.masks.device

    def nbytes(self) -> int:
        ts = [self.masks, self.dmins, self.dmaxs, self.dexps, self.nsamps, self.cams,
              self.z_surface, self.raw_masks]
        return sum(int(t.numel() * t.element_size()) for t in ts if t is not None)

    @classmethod
    def from_views(cls, views, dev=None, with_z=False):
        """Copy (ViewGeometry, ConfidenceMask) pairs into device planes.

        Each host map is uploaded straight into its slot of the padded device
        plane (no host-side packing pass).  Raises ValueError on a mask/view
        size mismatch (fusion.py:669-670).
        """
        import torch
        dev = dev or device()
        cams = [vg.camera for vg, _m in views]
        hm = max(int(c.height) for c in cams)
        wm = max(int(c.width) for c in cams)
        nv = len(views)
        sizes = []
        for vg, m in views:
            c = vg.camera
            mv = m.values if hasattr(m, "values") else np.asarray(m)
            if tuple(mv.shape) != (c.height, c.width):
                raise ValueError("mask and view dimensions differ")
            sizes.append((int(c.height), int(c.width)))
        alloc = torch.empty if all(s == (hm, wm) for s in sizes) else torch.zeros
        names = ["masks", "dmins", "dmaxs", "dexps", "nsamps"] + (["z_surface"] if with_z else [])
        planes = {k: alloc((nv, hm, wm), dtype=torch.int32 if k == "nsamps" else torch.float32,
                           device=dev) for k in names}
        from .staging import is_pinned, stager
        srcs = []
        for (vg, m), (h, w) in zip(views, sizes):
            src = {"masks": m.values if hasattr(m, "values") else m, "dmins": vg.d_min,
                   "dmaxs": vg.d_max, "dexps": vg.d_exp, "nsamps": vg.n_samples}
            if with_z:
                src["z_surface"] = vg.z_surface
            srcs.append({k: np.ascontiguousarray(src[k], np.int32 if k == "nsamps" else np.float32)
                         for k in names})
        # page-locked maps are DMA sources as they are; pageable ones (what
        # render_view returns) go through the pinned staging ring (host
        # threads + DMA) instead of torch's synchronous pageable copies
        pageable = [(i, k) for i in range(nv) for k in names if not is_pinned(srcs[i][k])]
        if pageable:
            cur = torch.cuda.current_stream(dev)
            with _device_lock(dev):
                stg = stager(dev)
                for i, k in pageable:
                    stg.copy2d(planes[k][i].data_ptr(), 4 * wm, srcs[i][k], cur)
                stg.flush()
        staged = set(pageable)
        for i, (h, w) in enumerate(sizes):
            for k in names:
                if (i, k) not in staged:
                    planes[k][i, :h, :w].copy_(torch.from_numpy(srcs[i][k]), non_blocking=True)
        cam_t = torch.from_numpy(pack_cameras(cams)).to(dev)
        torch.cuda.current_stream(dev).synchronize()   # the host maps may go after return
        return cls(cam_t, planes["masks"], planes["dmins"], planes["dmaxs"], planes["dexps"],
                   planes["nsamps"], z_surface=planes.get("z_surface"), sizes=sizes)

    def refine(self, raw_masks=None, stream=None):
        """Refine ``raw_masks`` (default: the stored raw masks) into ``masks`` on device."""
        from .segmenter import refine_masks_device
        raw = raw_masks if raw_masks is not None else self.raw_masks
        if raw is None or self.z_surface is None:
            raise ValueError("refine() needs raw masks and z_surface planes")
        refine_masks_device(raw, self.z_surface, self.nsamps, out=self.masks, stream=stream)
        return self


# ---------------------------------------------------------------------------
# the fusion operator
# ---------------------------------------------------------------------------

class Fuser:
    """Reusable device-side fusion of one grid layout with fixed parameters.

    ``run`` enqueues ``divas_fuse`` on the current stream (no host sync) and
    returns the device outputs.  ``vox_range`` restricts the call to a flat
    voxel range -- an axis-0 slab is ``[ix0 * G^2, ix1 * G^2)``.
    """

    def __init__(self, grid, params, bounds=None):
        self.grid = grid
        self.g = int(grid.resolution)
        self.origin = np.asarray(grid.origin, dtype=np.float64).reshape(3)
        self.dx = float(grid.voxel_size())
        self.pv = _params_vector(params)
        self.bc, self.bh, self.unb = bounds_arrays(bounds)
        self._cap_key = None
        self._cap = None

    def _args(self, density, lo, hi):
        a = _native.FuseArgs()
        a.g = self.g
        a.origin[:] = self.origin.tolist()
        a.dx_vox = self.dx
        a.density = _native.ptr(density)
        a.pv[:] = self.pv.tolist()
        a.bc[:] = self.bc.tolist()
        a.bh[:] = self.bh.tolist()
        a.unbounded = int(self.unb)
        a.vox_lo, a.vox_hi = lo, hi
        return a

    def capacity(self, density, lo, hi, stream=None) -> int:
        """Exact count of voxels passing the density gate in [lo, hi).

        One counting pass and one host sync per density tensor / range; the
        result sizes the workspace and is cached (keyed on the tensor's
        storage and version counter), so repeated fusions stay sync-free.
        """
        import ctypes
        import torch
        key = (density.data_ptr(), density._version, lo, hi, tuple(self.pv[[4, 5, 13]]))
        if self._cap_key != key:
            ws = torch.zeros(256, dtype=torch.uint8, device=density.device)
            a = self._args(density, lo, hi)
            _native.check(_native.lib().divas_gate_count(ctypes.byref(a), _native.ptr(ws),
                                                         _native.stream_handle(stream)),
                          "divas_gate_count")
            self._cap = int(ws[:8].view(torch.int64).item())
            self._cap_key = key
        return self._cap

    def run(self, density, views: DeviceViews, probs=None, stats=False, occ=False,
            occ_thr=0.5, vox_range=None, workspace=None, stream=None, max_gated=None,
            aux=None, nv_cap=None, incremental=None, steps=None, view_range=None,
            occ_peers=None, fallbacks=None):
        """Enqueue ``divas_fuse``.  ``aux``: ViewAux from ``refine_bands_device``
        (else built in the workspace).  ``incremental=(v0, v1)``: re-evaluate
        only views [v0, v1) against the state a previous full ``run`` left in
        ``workspace`` (same density, range, params and output buffers) --
        ``nv_cap`` sizes that workspace for views added later.  ``steps``:
        explicit ``_native.STEP_*`` flags with ``view_range`` (views-sharding).
        ``occ_peers``: (device pointer of an array of n buffer pointers, n) --
        the occupancy of the range is also stored into every listed [G^3]
        buffer (``sharding.PeerOccupancy``: the slab all-gather fused into the
        fusion's own stores over NVLink).  ``fallbacks``: a CUDA int64 tensor of
        ``_native.NFALLBACK`` counters that accumulate how often each certified
        shortcut handed a pair to the reference's exact chain
        (``_native.FALLBACKS`` names them)."""
        import ctypes
        import torch
        g = self.g
        nvox = g ** 3
        lo, hi = (0, nvox) if vox_range is None else (int(vox_range[0]), int(vox_range[1]))
        dev = views.device
        if density.dtype != torch.float32 or not density.is_cuda or density.numel() != nvox:
            raise ValueError("density must be a CUDA float32 tensor with G^3 entries")
        density = density.contiguous()
        cap = max_gated if max_gated is not None else self.capacity(density, lo, hi, stream)
        cap = max(int(cap), 1)
        if probs is None:
            probs = torch.empty(nvox, dtype=torch.float64, device=dev)
        elif probs is False:                  # GATE / PAIRS steps: no output grid
            probs = None
        out = {"probs": probs}
        if stats:
            out["n_thick"] = torch.empty(nvox, dtype=torch.int32, device=dev)
            out["n_thin"] = torch.empty(nvox, dtype=torch.int32, device=dev)
            for k in ("sw", "smw", "st"):
                out[k] = torch.empty(nvox, dtype=torch.float64, device=dev)
        if occ is True:
            out["occ"] = torch.empty(nvox, dtype=torch.uint8, device=dev)
        elif occ is not False and occ is not None:
            out["occ"] = occ
        lib = _native.lib()
        nvc = max(int(nv_cap or views.nv), views.nv)
        if hasattr(lib, "divas_fuse_workspace_size_ext"):
            wsb = lib.divas_fuse_workspace_size_ext(cap, nvc, views.hm, views.wm,
                                                    1 if aux is None else 0)
        else:                                   # experiment builds of older revisions
            wsb = lib.divas_fuse_workspace_size(cap, nvc, views.hm, views.wm)
        if workspace is None or workspace.numel() < wsb:
            workspace = torch.empty(wsb, dtype=torch.uint8, device=dev)
        out["workspace"] = workspace
        a = self._args(density, lo, hi)
        a.nv, a.hm, a.wm = views.nv, views.hm, views.wm
        a.cams = _native.ptr(views.cams)
        a.masks, a.dmins = _native.ptr(views.masks), _native.ptr(views.dmins)
        a.dmaxs, a.dexps = _native.ptr(views.dmaxs), _native.ptr(views.dexps)
        a.nsamps = _native.ptr(views.nsamps)
        a.probs = _native.ptr(probs)
        a.n_thick = _native.ptr(out.get("n_thick"))
        a.n_thin = _native.ptr(out.get("n_thin"))
        a.sw, a.smw, a.st = (_native.ptr(out.get(k)) for k in ("sw", "smw", "st"))
        a.occ = _native.ptr(out.get("occ"))
        a.occ_thr = float(occ_thr)
        a.max_gated = cap
        if aux is not None:
            a.records, a.bands = _native.ptr(aux.records), _native.ptr(aux.bands)
        a.nv_cap = nvc
        if occ_peers is not None:
            a.occ_peers, a.n_peers = int(occ_peers[0]), int(occ_peers[1])
        if fallbacks is not None:
            if (fallbacks.dtype != torch.int64 or not fallbacks.is_cuda or
                    fallbacks.numel() < _native.NFALLBACK):
                raise ValueError("fallbacks must be a CUDA int64 tensor of NFALLBACK counters")
            a.fallbacks = _native.ptr(fallbacks)
        if incremental is not None:
            a.mode = _native.FUSE_INCREMENTAL
            a.view_lo, a.view_hi = int(incremental[0]), int(incremental[1])
        elif steps is not None:
            a.mode = int(steps)
            v0, v1 = view_range if view_range is not None else (0, views.nv)
            a.view_lo, a.view_hi = int(v0), int(v1)
        _native.check(lib.divas_fuse(ctypes.byref(a), _native.ptr(workspace), wsb,
                                     _native.stream_handle(stream)), "divas_fuse")
        return out

    @staticmethod
    def gated_count(out) -> "torch.Tensor":
        """Device int64 scalar: voxels that cleared the density gate."""
        return out["workspace"][:8].view(__import__("torch").int64)

    @staticmethod
    def check_overflow(out):
        """Raise if the last run's workspace capacity was too small (syncs)."""
        import torch
        if int(out["workspace"][8:12].view(torch.int32).item()) != 0:
            raise RuntimeError("divas_fuse: gated voxels exceeded the workspace capacity")

    @staticmethod
    def gated_voxels(out, count=None):
        """Flat indices of the gated voxels (a superset of the nonzero p)."""
        import torch
        Fuser.check_overflow(out)
        n = int(Fuser.gated_count(out).item()) if count is None else int(count)
        ws = out["workspace"]
        return ws[256:256 + 4 * n].view(torch.int32).to(torch.int64) & 0xffffffff


def _upload_windows(lib, jobs, stream):
    """Window rectangles (src, dst, spitch, dpitch, width_bytes, rows) from
    page-locked host arrays: one ``divas_gather2d_h2d`` launch (the SMs read
    the rows through unified addressing; the copy engine moves short rows at
    a fraction of the link rate).  A source that is not page-locked makes the
    whole batch go through ``divas_copy2d_h2d`` instead (the gather validates
    every job before it launches)."""
    arr = (_native.Copy2D * len(jobs))(*[_native.Copy2D(*j) for j in jobs])
    h = _native.stream_handle(stream)
    if lib.divas_gather2d_h2d(arr, len(jobs), h) == 0:
        return
    for src, dst, sp, dp, wb, rows in jobs:
        _native.check(lib.divas_copy2d_h2d(dst, dp, src, sp, wb, rows, h), "divas_copy2d_h2d")


_ZERO_POOL = None


def _zeroed_host_async(nvox, threads=4):
    """A page-locked f64 buffer and the futures of its zero fill, run by
    ``threads`` host threads (libc memset through ctypes, GIL released) while
    the caller queues its uploads.  Few threads on purpose: the fill shares
    host memory bandwidth with the DMAs of the same update (16 threads slowed
    a concurrent 337 MB upload + 99 MB download by 0.7 ms, 4 by 0.3 ms).
    Wait on every future before the buffer is written."""
    import concurrent.futures as cf

    import torch
    global _ZERO_POOL
    if _ZERO_POOL is None:
        _ZERO_POOL = cf.ThreadPoolExecutor(max_workers=threads)
    host = torch.empty(nvox, dtype=torch.float64, pin_memory=True)
    base, n = host.data_ptr(), nvox * 8
    step = ((n + threads - 1) // threads + 4095) // 4096 * 4096   # page-aligned shares
    futs = [_ZERO_POOL.submit(ctypes.memset, base + o, 0, min(step, n - o))
            for o in range(0, n, step)] if n else []
    return host, futs


def _zeroed_host(nvox):
    """A zero-filled page-locked f64 buffer for the dense result.  Called while
    the device is still busy (uploads / fusion queued), so the parallel host
    fill overlaps the device work; the block returns to torch's host cache
    when the array built on it is released."""
    import torch
    host = torch.empty(nvox, dtype=torch.float64, pin_memory=True)
    host.zero_()
    return host


def _sparse_probs_to_host(out, nvox, host=None) -> np.ndarray:
    """Dense host probabilities from the gated list: only the gated voxels
    can be nonzero (the gate pass writes 0 everywhere else), so their (index,
    p) pairs are gathered on the device, copied, and scattered into a zeroed
    host buffer (``host``: from ``_zeroed_host``, filled while the device
    worked)."""
    import torch
    idx = Fuser.gated_voxels(out)
    vals = out["probs"].reshape(-1)[idx]
    if host is None:
        host = _zeroed_host(nvox)
    host[idx.cpu()] = vals.cpu()
    return host.numpy()


def _device_inputs(grid, density, views, params, bounds):
    _check_layout(grid, density)
    dev = device()
    dv = DeviceViews.from_views(views, dev)
    dens = _staged_to_device(density.values, np.float32, dev)
    return Fuser(grid, params, bounds), dens, dv


def fuse(grid, density, views, params, bounds=None, workers=None,
         trace_path=None) -> OccupancyGrid:
    """Fuse refined multi-view masks into an occupancy grid (fusion.py:692-724).

    ``views`` is a list of (ViewGeometry, ConfidenceMask) pairs.  ``workers``
    is accepted for signature compatibility and ignored (the kernel's result
    does not depend on it, as the reference's does not).  With ``trace_path``
    the GPU additionally records one JSON line per (voxel, view) decision.
    """
    g = int(grid.resolution)
    _check_layout(grid, density)
    if not views:
        return OccupancyGrid(grid, np.zeros((g, g, g)))
    if trace_path is not None:
        from .trace import fuse_traced
        return OccupancyGrid(grid, fuse_traced(grid, density, views, params, bounds, trace_path))
    fuser, dens, dv = _device_inputs(grid, density, views, params, bounds)
    out = fuser.run(dens, dv)
    host = _zeroed_host(g ** 3)
    return OccupancyGrid(grid, _sparse_probs_to_host(out, g ** 3, host).reshape(g, g, g))


def fuse_with_stats(grid, density, views, params, bounds=None):
    """``fuse`` plus the per-voxel integer votes and sorted sums."""
    g = int(grid.resolution)
    _check_layout(grid, density)
    if not views:
        z = np.zeros((g, g, g))
        zi = np.zeros((g, g, g), np.int32)
        return OccupancyGrid(grid, z), FusionStats(zi, zi.copy(), z, z.copy(), z.copy(), 0)
    fuser, dens, dv = _device_inputs(grid, density, views, params, bounds)
    out = fuser.run(dens, dv, stats=True)
    host = {k: out[k].cpu().numpy().reshape(g, g, g)
            for k in ("probs", "n_thick", "n_thin", "sw", "smw", "st")}
    gated = int(Fuser.gated_count(out).item())
    stats = FusionStats(host["n_thick"], host["n_thin"], host["sw"], host["smw"], host["st"],
                        gated)
    return OccupancyGrid(grid, host["probs"]), stats


def _trusted_mask(values):
    from .segmenter import trusted_mask
    return trusted_mask(values)


_STREAMS = {}


def _adjacent_run(arrs, dt, shape):
    """One (n, *shape) array over ``arrs`` when they are C-contiguous
    ``shape`` planes of dtype ``dt`` laid end to end in memory (e.g. slices of
    one stacked host buffer): one copy instead of n.  None otherwise."""
    first = arrs[0]
    if not isinstance(first, np.ndarray) or first.dtype != dt:
        return None
    nbytes = int(np.prod(shape)) * np.dtype(dt).itemsize
    base = first.__array_interface__["data"][0]
    for j, a in enumerate(arrs):
        if (not isinstance(a, np.ndarray) or a.dtype != dt or a.shape != tuple(shape) or
                not a.flags.c_contiguous or a.__array_interface__["data"][0] != base + j * nbytes):
            return None
    if len(arrs) == 1:
        return first.reshape((1,) + tuple(shape))
    buf = (ctypes.c_char * (nbytes * len(arrs))).from_address(base)
    return np.frombuffer(buf, dtype=dt).reshape((len(arrs),) + tuple(shape))


def _side_stream(dev, name):
    """A per-device side stream (uploads / downloads of the pipelined update)."""
    import torch
    key = (str(dev), name)
    if key not in _STREAMS:
        _STREAMS[key] = torch.cuda.Stream(device=dev)
    return _STREAMS[key]


_RF_LOCKS = {}
_RF_LOCKS_GUARD = __import__("threading").Lock()


class _device_lock:
    """Context manager: the per-device lock of the shared upload / download
    streams and the pinned staging ring (``refine_and_fuse``, ``fuse``'s view
    upload, ``project_grid_overlay``).  On an exception the staging ring's
    queued jobs are dropped, so none is issued later into released
    buffers."""

    def __init__(self, dev):
        key = str(dev)
        self.key = key
        with _RF_LOCKS_GUARD:
            self.lock = _RF_LOCKS.setdefault(key, __import__("threading").Lock())

    def __enter__(self):
        self.lock.acquire()
        return self

    def __exit__(self, exc_type, exc, tb):
        try:
            if exc_type is not None:
                from . import staging
                stg = staging._STAGERS.get(self.key)
                if stg is not None:
                    stg.discard()
        finally:
            self.lock.release()
        return False


def refine_and_fuse(grid, density, views, params, bounds=None, workers=None,
                    return_refined=True, chunk_views=4, windows=True, transfer_stats=None):
    with _device_lock(device()):
        return _refine_and_fuse(grid, density, views, params, bounds, workers, return_refined,
                                chunk_views, windows, transfer_stats)


def _refine_and_fuse(grid, density, views, params, bounds=None, workers=None,
                     return_refined=True, chunk_views=4, windows=True, transfer_stats=None):
    """``refine_mask`` on every (ViewGeometry, raw ConfidenceMask) pair, then
    ``fuse`` of the refined set -- the session's update (session.py:204-215)
    as one device pass: each host map is uploaded once, refinement writes the
    fusion's scan records directly.  Returns (OccupancyGrid, [refined
    ConfidenceMask] or None).

    Pipelined over chunks of ``chunk_views`` views: the planes upload on a
    side stream; each chunk is refined as soon as its full planes are in and
    its refined masks download on a second side stream while later planes
    still upload (the link is full duplex); its (view, voxel) pairs are
    evaluated (``divas_fuse`` PAIRS step for those views, current stream)
    once its depth-map windows are in.  After the last chunk
    only the value-sorted reduction and the (index, p) download of the gated
    voxels remain, so an update costs about the host-link time of its inputs.
    ``windows``: d_min / d_max are read by the fusion only at the centre
    pixels of gated voxels (and their neighbours), all inside each view's
    window around the projected gated region (``sharding.slab_view_rois``), so
    only those sub-rectangles are uploaded (C3: 49 % of the pixels).
    ``transfer_stats``: a dict that receives the bytes copied each way.

    Same validation and errors as the two reference calls; results identical
    to ``fuse(grid, density, [(v, refine_mask(m, v)) ...], params, bounds)``
    (the pair evaluations and the order-independent reduction do not depend
    on how the views are grouped).
    """
    import torch
    from .segmenter import (ViewAux, refine_bands_device, refine_masks_device,
                            refine_minmax_device)
    g = int(grid.resolution)
    nvox = g ** 3
    _check_layout(grid, density)
    views = list(views)
    for vg, m in views:
        if m.refined:
            raise ValueError("mask is already refined")
        if m.shape != vg.z_surface.shape:
            raise ValueError("mask and view dimensions differ")
    if not views:
        return OccupancyGrid(grid, np.zeros((g, g, g))), ([] if return_refined else None)
    dev = device()
    cur = torch.cuda.current_stream(dev)
    up, down = _side_stream(dev, "up"), _side_stream(dev, "down")
    fuser = Fuser(grid, params, bounds)
    cams = [vg.camera for vg, _m in views]
    nv = len(views)
    hm = max(int(c.height) for c in cams)
    wm = max(int(c.width) for c in cams)
    sizes = [(int(c.height), int(c.width)) for c in cams]
    alloc = torch.empty if all(sz == (hm, wm) for sz in sizes) else torch.zeros
    names = ("raw", "z", "dmins", "dmaxs", "dexps", "nsamps")
    planes = {k: alloc((nv, hm, wm), dtype=torch.int32 if k == "nsamps" else torch.float32,
                       device=dev) for k in names}
    aux = ViewAux.empty(nv, hm, wm, dev)
    keys_all = torch.empty((nv, 4), dtype=torch.int32, device=dev)
    refined = torch.empty((nv, hm, wm), dtype=torch.float32, device=dev) if return_refined else None
    host = (torch.empty((nv, hm, wm), dtype=torch.float32, pin_memory=True)
            if return_refined else None)
    cam_t = torch.from_numpy(pack_cameras(cams)).to(dev, non_blocking=True)
    # the result grid: page-locked, zero-filled by host threads from now on
    hp, hp_fill = _zeroed_host_async(nvox)
    try:
        # pageable host arrays (what render_view returns) go through pinned
        # staging slots filled by host threads (staging.Stager); pinned ones are
        # DMA sources as they are
        from .staging import is_pinned, stager
        first = views[0][1].values if hasattr(views[0][1], "values") else views[0][1]
        stg = None if is_pinned(first) else stager(dev)
        # 1. density first (the gate count needs it), then every view upload queued
        dvals = density.values
        if stg is not None and not isinstance(dvals, torch.Tensor) and not is_pinned(dvals):
            dens = torch.empty(nvox, dtype=torch.float32, device=dev)
            stg.copy(dens.data_ptr(), np.ascontiguousarray(dvals, np.float32), cur)
            stg.flush()
        else:
            dens = as_device(dvals, np.float32, dev, non_blocking=True)
        cnt = torch.zeros(256, dtype=torch.uint8, device=dev)
        _native.check(_native.lib().divas_gate_count(ctypes.byref(fuser._args(dens, 0, nvox)),
                                                     _native.ptr(cnt), _native.stream_handle()),
                      "divas_gate_count")
        up.wait_stream(cur)                       # planes allocated on the current stream
        chunk = max(1, int(chunk_views))
        bounds_k = [(v0, min(nv, v0 + chunk)) for v0 in range(0, nv, chunk)]
        ready = []
        srcs = [{"raw": m.values if hasattr(m, "values") else m, "z": vg.z_surface, "dmins": vg.d_min,
                 "dmaxs": vg.d_max, "dexps": vg.d_exp, "nsamps": vg.n_samples} for vg, m in views]

        h2d = [int(np.asarray(density.values).size) * 4]

        def upload_full(k, v0, v1):
            dt = np.int32 if k == "nsamps" else np.float32
            h2d[0] += sum(sizes[i][0] * sizes[i][1] for i in range(v0, v1)) * 4
            if stg is not None:
                for i in range(v0, v1):
                    stg.copy2d(planes[k][i].data_ptr(), 4 * wm,
                               np.ascontiguousarray(srcs[i][k], dt), up)
                return
            run = _adjacent_run([srcs[i][k] for i in range(v0, v1)], dt, (hm, wm))
            if run is not None:                   # the views' planes are one host block
                planes[k][v0:v1].copy_(torch.from_numpy(run), non_blocking=True)
                return
            for i in range(v0, v1):
                h, w = sizes[i]
                planes[k][i, :h, :w].copy_(torch.from_numpy(np.ascontiguousarray(srcs[i][k], dt)),
                                           non_blocking=True)

        # with windows, d_exp too is read only inside them (the band pass builds
        # records there; the planar refinement does not need it)
        full_names = ("raw", "z", "nsamps") if windows else ("raw", "z", "dexps", "nsamps")
        win_names = ("dmins", "dmaxs", "dexps") if windows else ("dmins", "dmaxs")
        full_ready = [None] * len(bounds_k)       # chunk c's full planes are on the device

        def upload_fulls(chunks):
            for c in chunks:
                v0, v1 = bounds_k[c]
                for k in full_names:
                    if k != "raw":
                        upload_full(k, v0, v1)
                if stg is not None:
                    stg.flush()
                full_ready[c] = torch.cuda.Event()
                full_ready[c].record(up)

        # Upload order: raw masks first (their per-view bounding box narrows the
        # depth maps' windows); the full z / n_samples planes of the first
        # chunks keep the link busy while the host waits for that box; then
        # every window, then the remaining full planes, so that each later
        # chunk's work can run as soon as its full planes land and the update
        # ends one chunk after the last upload.
        n_pre = min(2, len(bounds_k)) if windows else len(bounds_k)
        with torch.cuda.stream(up):
            for v0, v1 in bounds_k:
                upload_full("raw", v0, v1)
            if stg is not None:
                stg.flush()
            raw_done = torch.cuda.Event()
            raw_done.record(up)
            upload_fulls(range(n_pre))
        # the windows need the gated voxels' bounding box: one wait for the density
        # upload, while the full planes above keep the link busy
        rois = None
        lib = _native.lib()
        if windows:
            from .sharding import slab_view_rois
            rois = slab_view_rois(dens, fuser.pv, g, np.asarray(grid.origin, dtype=np.float64),
                                  fuser.dx, pack_cameras(cams), sizes)
            # d_min / d_max / d_exp are read only where the refined mask reaches
            # mask_thr or exceeds 0.5 (refined <= raw) and at those pixels'
            # 4-neighbours: intersect each window with the mask's box + 1 px
            thr = np.float32(min(float(fuser.pv[10]), 0.5))
            if float(thr) > min(float(fuser.pv[10]), 0.5):
                thr = np.nextafter(thr, np.float32(-np.inf))
            bbox = torch.empty((nv, 4), dtype=torch.int32, device=dev)
            cur.wait_event(raw_done)
            _native.check(lib.divas_mask_bbox(nv, hm, wm, planes["raw"].data_ptr(), float(thr),
                                              bbox.data_ptr(), _native.stream_handle()),
                          "divas_mask_bbox")
            mbox = bbox.cpu().numpy()
        keep = []
        # the last chunk's windows go after the remaining full planes, so that the
        # final upload is small and the refined masks of the last chunk download
        # while it streams (C3: 9.66 ms against 9.72-9.9 with none, 2 or 3)
        n_tail = 1 if windows and len(bounds_k) > n_pre else 0
        with torch.cuda.stream(up):
            for ci, (v0, v1) in enumerate(bounds_k):
                if ci == len(bounds_k) - n_tail:
                    upload_fulls(range(n_pre, len(bounds_k)))
                jobs = []                         # pinned sources: one gather launch per chunk
                for k in win_names:
                    if rois is None:
                        upload_full(k, v0, v1)
                        continue
                    for i in range(v0, v1):
                        h, w = sizes[i]
                        x0, y0, x1, y1 = (int(c) for c in rois.host[i])
                        x1, y1 = min(x1, w - 1), min(y1, h - 1)
                        bx0, by0, bx1, by1 = (int(c) for c in mbox[i])
                        if bx1 < 0:
                            continue                  # no pixel can need a depth value
                        x0, y0 = max(x0, bx0 - 1), max(y0, by0 - 1)
                        x1, y1 = min(x1, bx1 + 1), min(y1, by1 + 1)
                        if x1 < x0 or y1 < y0:
                            continue
                        a = np.ascontiguousarray(srcs[i][k], np.float32)
                        keep.append(a)
                        h2d[0] += 4 * (x1 - x0 + 1) * (y1 - y0 + 1)
                        if stg is not None:
                            stg.copy2d(planes[k][i].data_ptr() + 4 * (y0 * wm + x0), 4 * wm,
                                       a[y0:y1 + 1, x0:x1 + 1], up)
                            continue
                        jobs.append((a.ctypes.data + 4 * (y0 * w + x0),
                                     planes[k][i].data_ptr() + 4 * (y0 * wm + x0), 4 * w, 4 * wm,
                                     4 * (x1 - x0 + 1), y1 - y0 + 1))
                if jobs:
                    _upload_windows(lib, jobs, up)
                if stg is not None:
                    stg.flush()
                ev = torch.cuda.Event()
                ev.record(up)
                ready.append(ev)
            if n_tail == 0:
                upload_fulls(range(n_pre, len(bounds_k)))
        # 2. exact workspace size (the count finished long before the uploads)
        cap = max(int(cnt[:8].view(torch.int64).item()), 1)
        dv = DeviceViews(cam_t, refined if refined is not None else planes["raw"], planes["dmins"],
                         planes["dmaxs"], planes["dexps"], planes["nsamps"], sizes=sizes)
        # The result grid lives in page-locked host memory: zero-filled by the
        # host while the views upload, and the reduction writes the gated voxels'
        # p into it directly (unified addressing) -- no gather, copy or scatter.
        # The gate pass gets no output (probs=None) so it leaves the grid alone.
        kw = dict(max_gated=cap, aux=aux)
        out = fuser.run(dens, dv, steps=_native.STEP_GATE | _native.STEP_CLEAR_ALL, probs=False, **kw)
        kw["workspace"] = out["workspace"]
        # 3. per chunk: refine -> pairs of those views; refined masks download.
        # With windows the planar refinement needs only the full planes, so each
        # chunk's is queued behind them and its download overlaps the rest of
        # the uploads (the link is full duplex); the scan records / bands and the
        # pairs then wait for the chunk's windows.
        for c, ((v0, v1), ev) in enumerate(zip(bounds_k, ready)):
            if rois is not None:
                cur.wait_event(full_ready[c])
                keys = keys_all[v0:v1]
                if return_refined:
                    refine_masks_device(planes["raw"][v0:v1], planes["z"][v0:v1],
                                        planes["nsamps"][v0:v1], out=refined[v0:v1], keys=keys)
                    down.wait_stream(cur)
                    with torch.cuda.stream(down):
                        host[v0:v1].copy_(refined[v0:v1], non_blocking=True)
                else:
                    refine_minmax_device(planes["z"][v0:v1], planes["nsamps"][v0:v1], keys=keys)
            cur.wait_event(ev)
            if rois is not None:
                refine_bands_device(planes["raw"][v0:v1], planes["z"][v0:v1],
                                    planes["nsamps"][v0:v1], planes["dexps"][v0:v1], fuser.pv,
                                    fuser.dx, aux=aux.view_slices(v0, v1, nv, hm, wm), planar=False,
                                    roi=rois.subset(v0, v1), keys=keys)
            else:
                refine_bands_device(planes["raw"][v0:v1], planes["z"][v0:v1],
                                    planes["nsamps"][v0:v1], planes["dexps"][v0:v1], fuser.pv,
                                    fuser.dx, out=refined[v0:v1] if return_refined else None,
                                    aux=aux.view_slices(v0, v1, nv, hm, wm), planar=return_refined)
            fuser.run(dens, dv, steps=_native.STEP_PAIRS, view_range=(v0, v1), probs=False, **kw)
            if return_refined and rois is None:
                down.wait_stream(cur)
                with torch.cuda.stream(down):
                    host[v0:v1].copy_(refined[v0:v1], non_blocking=True)
        # 4. reduction (p lands in hp), then the overflow flag
        for f in hp_fill:                         # the zero fill ran beside the uploads
            f.result()
        fuser.run(dens, dv, steps=_native.STEP_REDUCE, probs=hp, **kw)
        hdr_h = torch.empty(16, dtype=torch.uint8, pin_memory=True)
        hdr_h.copy_(kw["workspace"][:16], non_blocking=True)
        cur.synchronize()
        if int(hdr_h[8:12].view(torch.int32).item()) != 0:
            raise RuntimeError("divas_fuse: gated voxels exceeded the workspace capacity")
        hpn = hp.numpy()
        if transfer_stats is not None:
            transfer_stats["h2d_bytes"] = h2d[0] + cam_t.numel() * 8
            # the header, each gated voxel's p (stored into the host grid by the
            # reduction) and the refined masks
            transfer_stats["d2h_bytes"] = 16 + 8 * cap + (sum(h * w for h, w in sizes) * 4
                                                          if return_refined else 0)
        masks = None
        if return_refined:
            down.synchronize()
            hn = host.numpy()
            masks = [_trusted_mask(hn[i, :h, :w]) for i, (h, w) in enumerate(sizes)]
        return OccupancyGrid(grid, hpn.reshape(g, g, g)), masks
    finally:
        for f in hp_fill:                     # never leave a fill writing into a freed block
            f.result()


refine_and_fuse.__doc__ = (_refine_and_fuse.__doc__ or "") + """
    Calls on one device are serialised (they share its upload / download
    streams and pinned staging ring), so callers on several threads -- the
    reference's service fuses concurrently across sessions (service.py:88-94)
    -- stay correct.
    """


def gradient_maps_device(views: DeviceViews, eps: float, kappa: float, stream=None):
    """f64 depth-gradient maps on the padded planes (fusion._gradient_maps)."""
    import torch
    out = torch.empty(views.masks.shape, dtype=torch.float64, device=views.device)
    lib = _native.lib()
    _native.check(lib.divas_gradient_maps(views.nv, views.hm, views.wm,
                                          _native.ptr(views.dexps), _native.ptr(views.dmins),
                                          _native.ptr(views.dmaxs), _native.ptr(views.nsamps),
                                          float(eps), float(kappa), 1, _native.ptr(out),
                                          _native.stream_handle(stream)), "divas_gradient_maps")
    return out


# ---------------------------------------------------------------------------
# threshold / extract  (kernel (c))
# ---------------------------------------------------------------------------

def threshold_device(probs, thr=0.5, g=0, want_indices=False, stream=None):
    """``probs >= thr`` on device; optionally the C-order indices too.

    Returns (occ uint8 tensor, idx int64 tensor or None, count int64 tensor).
    ``idx`` rows are (ix, iy, iz) when ``g > 0`` (np.argwhere of the (G,G,G)
    grid), flat indices otherwise; only the first ``count`` rows are valid.
    """
    import torch
    p = probs.reshape(-1)
    if p.dtype != torch.float64 or not p.is_cuda:
        raise ValueError("threshold_device expects a CUDA float64 tensor")
    p = p.contiguous()
    n = p.numel()
    dev = p.device
    occ = torch.empty(n, dtype=torch.uint8, device=dev)
    cnt = torch.zeros(1, dtype=torch.int64, device=dev)
    idx = None
    if want_indices:
        idx = torch.empty((n, 3) if g > 0 else (n,), dtype=torch.int64, device=dev)
    lib = _native.lib()
    wsb = lib.divas_threshold_workspace_size(n)
    ws = torch.empty(wsb, dtype=torch.uint8, device=dev)
    _native.check(lib.divas_threshold(_native.ptr(p), n, float(thr), int(g), _native.ptr(occ),
                                      _native.ptr(idx), _native.ptr(cnt), _native.ptr(ws), wsb,
                                      _native.stream_handle(stream)), "divas_threshold")
    return occ, idx, cnt


def extract_device(probs, thr=0.5, stream=None):
    """Device ``np.argwhere(probs >= thr)`` of a (G,G,G) CUDA f64 grid.

    Returns (idx (G^3, 3) int64 tensor, count int64 tensor); rows past
    ``count`` are unspecified.  No host synchronisation.
    """
    g = int(probs.shape[0])
    _occ, idx, cnt = threshold_device(probs, thr, g=g, want_indices=True, stream=stream)
    return idx, cnt


def _as_probs_tensor(probs):
    import torch
    if isinstance(probs, torch.Tensor) and probs.is_cuda:
        return probs, True
    return as_device(np.asarray(probs), np.float64, device()), False


def threshold(probs, thr: float = 0.5):
    """Binary occupancy ``probs >= thr`` (ablation.py:109); same shape as probs."""
    p, on_dev = _as_probs_tensor(probs)
    occ, _idx, _cnt = threshold_device(p, thr)
    occ = occ.reshape(p.shape).bool()
    return occ if on_dev else occ.cpu().numpy()


def extract(probs, thr: float = 0.5):
    """``np.argwhere(probs >= thr)`` for a (G, G, G) grid: (N, 3) int64, C order."""
    p, on_dev = _as_probs_tensor(probs)
    if p.dim() != 3 or not (p.shape[0] == p.shape[1] == p.shape[2]):
        raise ValueError("extract expects a (G, G, G) probability grid")
    _occ, idx, cnt = threshold_device(p, thr, g=int(p.shape[0]), want_indices=True)
    n = int(cnt.item())
    idx = idx[:n]
    return idx if on_dev else idx.cpu().numpy()


# ---------------------------------------------------------------------------
# overlay (fusion.py:846-865)
# ---------------------------------------------------------------------------

def project_grid_overlay_device(probs, grid, camera, d_min, d_max, n_samples,
                                threshold: float = 0.5, bounds=None, out=None, stream=None):
    """``project_grid_overlay`` on device-resident data: ``probs`` the fused
    [G^3] f64 grid and the view's (H, W) d_min / d_max / n_samples as CUDA
    tensors; returns the (H, W) uint8 overlay on the device (no host sync)."""
    import ctypes
    h, w = int(camera.height), int(camera.width)
    if out is None:
        out = empty((h, w), np.uint8, probs.device)
    rec = pack_cameras([camera])[0]
    bc, bh, unb = bounds_arrays(bounds)
    D3 = ctypes.c_double * 3
    origin = np.asarray(grid.origin, dtype=np.float64).reshape(3)
    _native.check(_native.lib().divas_overlay(
        rec.ctypes.data_as(ctypes.c_void_p), h, w, _native.ptr(d_min), _native.ptr(d_max),
        _native.ptr(n_samples), _native.ptr(probs.contiguous()), int(grid.resolution),
        D3(*origin), float(grid.voxel_size()), D3(*bc), D3(*bh), int(unb), float(threshold),
        _native.ptr(out), _native.stream_handle(stream)), "divas_overlay")
    return out


def _staged_to_device(arr, np_dtype, dev):
    """A large host array (the dense grid, the density) on the device.  A
    pageable numpy array goes through the pinned staging ring
    (``staging.Stager``, host threads + DMA) instead of torch's synchronous
    pageable copy (~10 GB/s); page-locked arrays (what ``fuse`` /
    ``refine_and_fuse`` return) and torch tensors are copied directly."""
    import torch

    from .staging import is_pinned, stager
    if isinstance(arr, torch.Tensor):
        return as_device(arr, np_dtype, dev)
    a = np.ascontiguousarray(arr, dtype=np_dtype)
    pinned = is_pinned(a)
    if a.nbytes < (16 << 20) or pinned:
        t = as_device(a, np_dtype, dev, non_blocking=pinned)
        if pinned:
            torch.cuda.current_stream(dev).synchronize()   # `a` may go after return
        return t
    t = empty(a.shape, np_dtype, dev)
    with _device_lock(dev):                   # one user of the staging ring at a time
        stg = stager(dev)
        stg.copy(t.data_ptr(), a, torch.cuda.current_stream(dev))
        stg.flush()                           # host copies done: `a` may go
    return t


def project_grid_overlay(ogrid: OccupancyGrid, view, threshold: float = 0.5,
                         bounds=None) -> np.ndarray:
    """Binary (H, W) mask of pixels whose ray meets a voxel with p >= threshold
    (fusion.py:846-865)."""
    dev = device()
    p = _staged_to_device(ogrid.probs, np.float64, dev)
    dmin = as_device(view.d_min, np.float32, dev)
    dmax = as_device(view.d_max, np.float32, dev)
    ns = as_device(view.n_samples, np.int32, dev)
    out = project_grid_overlay_device(p, ogrid.grid, view.camera, dmin, dmax, ns, threshold,
                                      bounds)
    return out.cpu().numpy().astype(bool)
