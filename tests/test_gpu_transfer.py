"""Host -> device window uploads: ``divas_gather2d_h2d`` (the SMs read the
rows of page-locked host arrays) equals one ``divas_copy2d_h2d`` per window
byte for byte, at every alignment of the window's first column; a pageable
source is refused with DIVAS_EINVAL before anything launches, and
``refine_and_fuse``'s window upload then takes the copy-engine path."""

import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def _pinned(shape, rng):
    import torch
    t = torch.empty(shape, dtype=torch.float32, pin_memory=True)
    a = t.numpy()
    a[...] = rng.random(shape, dtype=np.float32) + 1.0
    return t, a


# w = 203: host pitch 812 B against 832 B on the device (rows mostly take the
# byte path); w = 208: both pitches 832 B (16-byte body, ragged ends);
# 130 jobs: more than one launch batch
@pytest.mark.parametrize("n_jobs,w", [(1, 203), (7, 208), (130, 203), (130, 208)])
def test_gather_equals_copy2d(n_jobs, w):
    import torch
    from paper_2601_04860_b200 import _native
    lib = _native.lib()
    dev = torch.device("cuda", 0)
    rng = np.random.default_rng(1000 + n_jobs)
    h, wm = 97, 208
    keep, jobs = [], []
    dst_a = torch.zeros((n_jobs, h, wm), dtype=torch.float32, device=dev)
    dst_b = torch.zeros_like(dst_a)
    for j in range(n_jobs):
        t, a = _pinned((h, w), rng)
        keep.append(t)
        x0 = int(rng.integers(0, w)); x1 = int(rng.integers(x0, w))
        y0 = int(rng.integers(0, h)); y1 = int(rng.integers(y0, h))
        if j == 0:
            x0, x1, y0, y1 = 0, w - 1, 0, h - 1                  # a whole plane
        if j == 1:
            x1 = x0                                             # one column
        jobs.append((a.ctypes.data + 4 * (y0 * w + x0), dst_a[j].data_ptr() + 4 * (y0 * wm + x0),
                     4 * w, 4 * wm, 4 * (x1 - x0 + 1), y1 - y0 + 1))
    arr = (_native.Copy2D * n_jobs)(*[_native.Copy2D(*jb) for jb in jobs])
    s = _native.stream_handle()
    assert lib.divas_gather2d_h2d(arr, n_jobs, s) == 0, lib.divas_last_error()
    for (src, _d, sp, dp, wb, rows), j in zip(jobs, range(n_jobs)):
        off = _d - dst_a[j].data_ptr()
        assert lib.divas_copy2d_h2d(dst_b[j].data_ptr() + off, dp, src, sp, wb, rows, s) == 0
    torch.cuda.synchronize()
    assert torch.equal(dst_a.view(torch.int32), dst_b.view(torch.int32))
    assert int(dst_a.view(torch.int32).count_nonzero()) > 0


def test_gather_refuses_pageable_source():
    import torch
    from paper_2601_04860_b200 import _native
    lib = _native.lib()
    a = np.ones((8, 8), np.float32)                          # ordinary numpy
    d = torch.zeros((8, 8), dtype=torch.float32, device="cuda")
    job = (_native.Copy2D * 1)(_native.Copy2D(a.ctypes.data, d.data_ptr(), 32, 32, 32, 8))
    assert lib.divas_gather2d_h2d(job, 1, _native.stream_handle()) == 1      # DIVAS_EINVAL
    assert b"page-locked" in lib.divas_last_error()
    torch.cuda.synchronize()
    assert float(d.abs().sum()) == 0.0


def test_upload_windows_falls_back_for_pageable():
    import torch
    from paper_2601_04860_b200 import _native
    from paper_2601_04860_b200.fusion import _upload_windows
    lib = _native.lib()
    a = np.arange(64, dtype=np.float32).reshape(8, 8)
    d = torch.zeros((8, 8), dtype=torch.float32, device="cuda")
    _upload_windows(lib, [(a.ctypes.data + 4 * 9, d.data_ptr() + 4 * 9, 32, 32, 12, 5)],
                    torch.cuda.current_stream())
    torch.cuda.synchronize()
    ref = np.zeros((8, 8), np.float32)
    ref[1:6, 1:4] = a[1:6, 1:4]
    assert np.array_equal(d.cpu().numpy(), ref)


def test_stager_discard_drops_queued_jobs():
    """After an error the lock holder drops the staging ring's queued jobs:
    none is issued later (into a buffer the failed caller released)."""
    import torch
    from paper_2601_04860_b200 import fusion, staging
    dev = torch.device("cuda", 0)
    stg = staging.stager(dev)
    dst = torch.zeros(1 << 20, dtype=torch.float32, device=dev)
    src = np.ones(1 << 20, np.float32)
    with pytest.raises(RuntimeError):
        with fusion._device_lock(dev):
            stg.copy(dst.data_ptr(), src, torch.cuda.current_stream(dev))
            raise RuntimeError("caller failed before flush")
    assert not stg.pending
    stg.flush()
    torch.cuda.synchronize()
    # whatever the ring issued before the error, nothing is issued after it;
    # and the ring still works
    dst2 = torch.zeros(1 << 20, dtype=torch.float32, device=dev)
    with fusion._device_lock(dev):
        stg.copy(dst2.data_ptr(), src, torch.cuda.current_stream(dev))
        stg.flush()
    torch.cuda.synchronize()
    assert float(dst2.sum()) == float(1 << 20)


def test_staged_api_uploads_match_device_inputs():
    """The drop-in APIs' large pageable inputs go through the staging ring
    (fusion._staged_to_device: >= 16 MiB): fuse() with a 168^3 pageable
    density and project_grid_overlay() with a 128^3 pageable grid give the
    same bits as the same data handed over as CUDA tensors."""
    import torch
    from paper_2601_04860_b200 import (DensityGrid, FusionParams, OccupancyGrid, VoxelGrid,
                                       fuse, project_grid_overlay, project_grid_overlay_device)
    from paper_2601_04860_b200.fusion import DeviceViews, Fuser
    from tests import golden_io
    from tests.gpu_cases import reference_objects
    case = golden_io.scene_cases()["sop"]
    grid0, _d, views, bounds = reference_objects(case)
    rng = np.random.default_rng(5)
    g = 168                                            # 18.9 MB of f32 density
    grid = VoxelGrid(g, grid0.half_extent, grid0.origin)
    dens = rng.random((g, g, g), dtype=np.float32) * 6.0
    dens[dens < 4.5] = 0.0                             # ~25 % gated
    og = fuse(grid, DensityGrid(grid, dens), views, FusionParams(), bounds=bounds)
    dev = torch.device("cuda", 0)
    dv = DeviceViews.from_views(views, dev)
    out = Fuser(grid, FusionParams(), bounds).run(torch.from_numpy(dens.reshape(-1)).to(dev), dv)
    ref = out["probs"].cpu().numpy().reshape(g, g, g)
    assert np.array_equal(og.probs, ref)
    assert int((ref > 0).sum()) > 0
    # overlay of a 128^3 grid (16 MiB of f64): pageable numpy vs CUDA tensor
    g2 = 128
    grid2 = VoxelGrid(g2, grid0.half_extent, grid0.origin)
    p = rng.random((g2, g2, g2))
    vg = views[0][0]
    got = project_grid_overlay(OccupancyGrid(grid2, p), vg, threshold=0.97)
    t = lambda a: torch.from_numpy(np.ascontiguousarray(a)).to(dev)   # noqa: E731
    want = project_grid_overlay_device(t(p.reshape(-1)), grid2, vg.camera, t(vg.d_min),
                                       t(vg.d_max), t(vg.n_samples), 0.97)
    want = want.cpu().numpy().astype(bool)
    assert np.array_equal(got, want) and got.any() and not got.all()


def test_gather_empty_jobs_are_noops():
    """No jobs, zero rows or zero width: nothing launched, success."""
    import torch
    from paper_2601_04860_b200 import _native
    lib = _native.lib()
    s = _native.stream_handle()
    assert lib.divas_gather2d_h2d(None, 0, s) == 0
    t = torch.empty(64, dtype=torch.float32, pin_memory=True)
    d = torch.full((64,), 3.0, dtype=torch.float32, device="cuda")
    jobs = (_native.Copy2D * 2)(_native.Copy2D(t.data_ptr(), d.data_ptr(), 256, 256, 0, 4),
                                _native.Copy2D(t.data_ptr(), d.data_ptr(), 256, 256, 64, 0))
    assert lib.divas_gather2d_h2d(jobs, 2, s) == 0
    torch.cuda.synchronize()
    assert float(d.min()) == 3.0 and float(d.max()) == 3.0
    bad = (_native.Copy2D * 1)(_native.Copy2D(t.data_ptr(), d.data_ptr(), 16, 16, 64, 1))
    assert lib.divas_gather2d_h2d(bad, 1, s) == 1            # width beyond the pitches
