"""Depth-weighted confidence refinement on the B200 (stage (a) of the path).

Drop-in for ``divas.segmenter.refine_mask`` / ``ConfidenceMask``
(/root/reference/pkg/src/divas/segmenter.py:46-62, :129-152): same signature,
same validation and error types, bit-identical float32 output.  The work runs
in ``divas_refine`` (csrc/refine.cu); there is no CPU path.
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np

from . import _native
from ._device import as_device, device, empty

__all__ = ["ConfidenceMask", "ViewAux", "ViewWindows", "refine_mask", "refine_masks",
           "refine_masks_device", "refine_bands_device", "refine_minmax_device"]


@dataclass
class ConfidenceMask:
    """Per-pixel segmentation confidence in [0, 1] (segmenter.py:46-62)."""

    values: np.ndarray  # (H, W) float32
    refined: bool = False

    def __post_init__(self):
        self.values = np.asarray(self.values, dtype=np.float32)
        if self.values.ndim != 2:
            raise ValueError("mask must be 2D")
        if self.values.size and (self.values.min() < 0 or self.values.max() > 1):
            raise ValueError("mask confidences must lie in [0, 1]")

    @property
    def shape(self):
        return self.values.shape


def trusted_mask(values) -> ConfidenceMask:
    """A refined ConfidenceMask built from kernel output, skipping the host
    range scan of ``__post_init__``: the refinement clips to [0, 1] (NaN
    passes the reference's scan too), so the scan cannot fail (a 762 K-pixel
    view: ~0.4 ms of host time per mask)."""
    m = ConfidenceMask.__new__(ConfidenceMask)
    m.values = values
    m.refined = True
    return m


def refine_masks_device(masks, z_surface, n_samples, out=None, stream=None, keys=None):
    """Batched refinement of device-resident planes ``[nv, hm, wm]``.

    ``masks``/``z_surface`` float32, ``n_samples`` int32 (CUDA tensors, C
    order).  Each view is normalised over its own valid pixels (padding with
    ``n_samples == 0`` is ignored and comes out as 0).  Returns ``out``.
    ``keys``: an int32 [nv, 4] CUDA tensor that receives the views' refine
    keys (as ``refine_minmax_device``), e.g. for ``refine_bands_device(keys=)``.
    """
    import torch
    if masks.dim() == 2:
        masks, z_surface, n_samples = masks[None], z_surface[None], n_samples[None]
        if out is not None:
            out = out[None]
    nv, hm, wm = masks.shape
    if z_surface.shape != masks.shape or n_samples.shape != masks.shape:
        raise ValueError("mask and view dimensions differ")
    for t, dt in ((masks, torch.float32), (z_surface, torch.float32), (n_samples, torch.int32)):
        if t.dtype != dt or not t.is_cuda or not t.is_contiguous():
            raise ValueError("refine_masks_device expects contiguous CUDA float32/int32 planes")
    if out is None:
        out = torch.empty_like(masks)
    lib = _native.lib()
    wsb = lib.divas_refine_workspace_size(nv)
    if keys is not None:
        if keys.numel() * keys.element_size() < wsb or not keys.is_cuda:
            raise ValueError("keys must be a CUDA int32 [nv, 4] tensor")
        ws = keys
    else:
        ws = torch.empty(wsb, dtype=torch.uint8, device=masks.device)
    _native.check(lib.divas_refine(nv, hm, wm, _native.ptr(masks), _native.ptr(z_surface),
                                   _native.ptr(n_samples), _native.ptr(out), _native.ptr(ws),
                                   wsb, _native.stream_handle(stream)), "divas_refine")
    return out


class ViewAux:
    """The fusion's per-view auxiliary data (csrc/bands.cuh), device-resident:
    ``records`` (per view two float2 planes: {refined mask, d_exp or NaN},
    {tau, n_samples}) and ``bands`` (per view the 8x8-tile depth bands and the
    view's tau range), as bytes.
    Built by ``refine_bands_device`` for given FusionParams / voxel size."""

    def __init__(self, records, bands):
        self.records = records
        self.bands = bands

    @classmethod
    def empty(cls, nv, hm, wm, dev):
        import torch
        lib = _native.lib()
        return cls(torch.empty(lib.divas_records_size(nv, hm, wm), dtype=torch.uint8, device=dev),
                   torch.empty(lib.divas_bands_size(nv, hm, wm), dtype=torch.uint8, device=dev))

    def view_slices(self, v0, v1, nv, hm, wm):
        """(records, bands) byte views of views [v0, v1)."""
        lib = _native.lib()
        r1 = lib.divas_records_size(1, hm, wm)
        b1 = lib.divas_bands_size(1, hm, wm)
        return self.records[v0 * r1: v1 * r1], self.bands[v0 * b1: v1 * b1]


def refine_minmax_device(z_surface, n_samples, keys=None, stream=None):
    """Per-view z min / max (order-preserving uint32 keys) and n min / max over
    valid pixels, [nv, 4] (int32 tensor view), for
    ``refine_bands_device(keys=...)``; the
    views of a block can be computed on one rank and the keys all-gathered."""
    import torch
    nv, hm, wm = z_surface.shape
    if keys is None:
        keys = torch.empty((nv, 4), dtype=torch.int32, device=z_surface.device)
    _native.check(_native.lib().divas_refine_minmax(nv, hm, wm, _native.ptr(z_surface),
                                                    _native.ptr(n_samples), _native.ptr(keys),
                                                    _native.stream_handle(stream)),
                  "divas_refine_minmax")
    return keys


def refine_bands_device(masks, z_surface, n_samples, d_exp, params, voxel_size, out=None,
                        aux=None, stream=None, planar=True, roi=None, keys=None):
    """``refine_masks_device`` fused with the fusion's per-view aux data.

    One pass over the planes writes the refined masks (``planar=True``) and
    the ``ViewAux`` (scan records + tile depth bands) that ``Fuser.run(aux=)``
    consumes, so the fusion never re-reads the planar masks.  ``aux`` may be
    a preallocated ViewAux or a pair of byte tensors (records, bands) for a
    slice of a larger set.  ``keys``: the views' min/max keys from
    ``refine_minmax_device`` (skips the min/max pass).  ``roi``: a
    ``ViewWindows`` -- build records and
    bands only inside one window per view (``divas_refine_bands_roi``; the
    planar output, if any, is also written only there).  Returns (out or
    None, aux).
    """
    import ctypes
    import torch
    nv, hm, wm = masks.shape
    for t in (z_surface, n_samples, d_exp):
        if t.shape != masks.shape:
            raise ValueError("mask and view dimensions differ")
    for t, dt in ((masks, torch.float32), (z_surface, torch.float32), (n_samples, torch.int32),
                  (d_exp, torch.float32)):
        if t.dtype != dt or not t.is_cuda or not t.is_contiguous():
            raise ValueError("refine_bands_device expects contiguous CUDA float32/int32 planes")
    pv = np.asarray(params.as_vector() if hasattr(params, "as_vector") else params, np.float64)
    if out is None and planar:
        out = torch.empty_like(masks)
    if not planar:
        out = None
    lib = _native.lib()
    if aux is None:
        aux = ViewAux.empty(nv, hm, wm, masks.device)
    rec, bands = (aux.records, aux.bands) if isinstance(aux, ViewAux) else aux
    if rec.numel() < lib.divas_records_size(nv, hm, wm) or \
            bands.numel() < lib.divas_bands_size(nv, hm, wm):
        raise ValueError("view aux buffers too small")
    wsb = lib.divas_refine_workspace_size(nv)
    ws = torch.empty(wsb, dtype=torch.uint8, device=masks.device)
    pvc = (ctypes.c_double * 14)(*pv.tolist())
    if keys is not None:
        if keys.numel() < 4 * nv or keys.dtype != torch.int32 or not keys.is_cuda:
            raise ValueError("keys must be a CUDA int32 [nv, 4] tensor")
        _native.check(lib.divas_refine_bands_keys(
            nv, hm, wm, _native.ptr(masks), _native.ptr(z_surface), _native.ptr(n_samples),
            _native.ptr(d_exp), _native.ptr(out), pvc, float(voxel_size), _native.ptr(rec),
            _native.ptr(bands), _native.ptr(keys), _native.ptr(ws), wsb,
            _native.ptr(roi.rects) if roi is not None else None,
            roi.max_w if roi is not None else 0, roi.max_h if roi is not None else 0,
            _native.stream_handle(stream)), "divas_refine_bands_keys")
        return out, aux
    if roi is not None:
        if roi.nv != nv:
            raise ValueError("one window per view")
        _native.check(lib.divas_refine_bands_roi(
            nv, hm, wm, _native.ptr(masks), _native.ptr(z_surface), _native.ptr(n_samples),
            _native.ptr(d_exp), _native.ptr(out), pvc, float(voxel_size), _native.ptr(rec),
            _native.ptr(bands), _native.ptr(ws), wsb, _native.ptr(roi.rects), roi.max_w,
            roi.max_h, _native.stream_handle(stream)), "divas_refine_bands_roi")
        return out, aux
    _native.check(lib.divas_refine_bands(nv, hm, wm, _native.ptr(masks), _native.ptr(z_surface),
                                         _native.ptr(n_samples), _native.ptr(d_exp),
                                         _native.ptr(out), pvc, float(voxel_size),
                                         _native.ptr(rec), _native.ptr(bands), _native.ptr(ws), wsb,
                                         _native.stream_handle(stream)), "divas_refine_bands")
    return out, aux


class ViewWindows:
    """One pixel window per view ({x0, y0, x1, y1}, inclusive, x0 / y0 on the
    8-pixel tile grid) on the device, for ``refine_bands_device(roi=...)``."""

    def __init__(self, rects, dev):
        import torch
        r = np.ascontiguousarray(np.asarray(rects, dtype=np.int32).reshape(-1, 4))
        if (r[:, 0] % 8).any() or (r[:, 1] % 8).any() or (r[:, 2] < r[:, 0]).any() or \
                (r[:, 3] < r[:, 1]).any():
            raise ValueError("windows must be non-empty and start on the 8-pixel tile grid")
        self.host = r
        self.nv = int(r.shape[0])
        self.max_w = int((r[:, 2] - r[:, 0] + 1).max())
        self.max_h = int((r[:, 3] - r[:, 1] + 1).max())
        self.rects = torch.from_numpy(r).to(dev)

    def subset(self, v0: int, v1: int) -> "ViewWindows":
        """The windows of views [v0, v1) (shares the device rectangles)."""
        w = ViewWindows.__new__(ViewWindows)
        w.host = self.host[v0:v1]
        w.nv = v1 - v0
        w.max_w = int((w.host[:, 2] - w.host[:, 0] + 1).max())
        w.max_h = int((w.host[:, 3] - w.host[:, 1] + 1).max())
        w.rects = self.rects[v0:v1]
        return w

    def fraction(self, hm: int, wm: int) -> float:
        """Share of the padded pixels inside the windows."""
        a = (np.minimum(self.host[:, 2], wm - 1) - self.host[:, 0] + 1) * \
            (np.minimum(self.host[:, 3], hm - 1) - self.host[:, 1] + 1)
        return float(a.sum()) / float(self.nv * hm * wm)


def refine_mask(mask: ConfidenceMask, view) -> ConfidenceMask:
    """Depth-weight a confidence mask by one minus the normalised depth.

    Same contract as the reference (segmenter.py:129-152): rejects refined
    masks and shape mismatches with ValueError; returns a new refined mask.
    """
    if mask.refined:
        raise ValueError("mask is already refined")
    if mask.shape != view.z_surface.shape:
        raise ValueError("mask and view dimensions differ")
    dev = device()
    m = as_device(mask.values, np.float32, dev)
    z = as_device(view.z_surface, np.float32, dev)
    n = as_device(view.n_samples, np.int32, dev)
    out = empty(m.shape, np.float32, dev)
    refine_masks_device(m, z, n, out=out)
    return trusted_mask(out.cpu().numpy())


def refine_masks(masks, views):
    """Batched ``refine_mask``: one upload, one launch, one download for all views.

    Same per-view validation and result as calling ``refine_mask`` on each
    (mask, view) pair; views of different sizes are padded on the device.
    """
    import torch
    masks, views = list(masks), list(views)
    if len(masks) != len(views):
        raise ValueError("need one view per mask")
    if not masks:
        return []
    for m, v in zip(masks, views):
        if m.refined:
            raise ValueError("mask is already refined")
        if m.shape != v.z_surface.shape:
            raise ValueError("mask and view dimensions differ")
    dev = device()
    hm = max(m.shape[0] for m in masks)
    wm = max(m.shape[1] for m in masks)
    nv = len(masks)
    same = all(m.shape == (hm, wm) for m in masks)
    alloc = torch.empty if same else torch.zeros
    M = alloc((nv, hm, wm), dtype=torch.float32, device=dev)
    Z = alloc((nv, hm, wm), dtype=torch.float32, device=dev)
    N = alloc((nv, hm, wm), dtype=torch.int32, device=dev)
    for i, (m, v) in enumerate(zip(masks, views)):
        h, w = m.shape
        M[i, :h, :w].copy_(torch.from_numpy(np.ascontiguousarray(m.values, np.float32)))
        Z[i, :h, :w].copy_(torch.from_numpy(np.ascontiguousarray(v.z_surface, np.float32)))
        N[i, :h, :w].copy_(torch.from_numpy(np.ascontiguousarray(v.n_samples, np.int32)))
    out = refine_masks_device(M, Z, N)
    host = out.cpu().numpy()
    return [trusted_mask(host[i, :m.shape[0], :m.shape[1]])
            for i, m in enumerate(masks)]
