"""Host -> device uploads of PAGEABLE host arrays through pinned staging slots.

The drop-in callers hand the fusion ordinary numpy arrays (``render_view``
returns them; /root/reference/pkg/src/divas/session.py:204-215).  A DMA from
pageable memory goes through the driver's own bounce buffer and serialises
with the host thread (~10 GB/s on the B200 boxes); ``refine_and_fuse``'s
pipelined update is then bound by it (C3: 53 ms against 10.6 ms from pinned
buffers).  ``Stager`` restores the pipeline: host worker threads copy chunks
of the source arrays into a ring of page-locked slots (numpy copies release
the GIL, so several run at once) while the copy engine moves earlier slots to
the device on the caller's stream (``divas_copy2d_h2d``).  A slot is refilled
only after the event of its previous DMA completed.

Jobs are contiguous copies or pitched 2-D windows (the depth-map windows of
``refine_and_fuse``); each is split into slot-sized chunks of whole rows.
"""

from __future__ import annotations

import collections
import concurrent.futures as cf
import os
import threading

import numpy as np

from . import _native

__all__ = ["Stager", "stager", "is_pinned"]


def is_pinned(a) -> bool:
    """True when ``a`` (numpy) lives in page-locked host memory (a DMA source
    as is)."""
    import torch
    try:
        return bool(torch.from_numpy(np.asarray(a)).is_pinned())
    except Exception:  # noqa: BLE001  (non-numpy-compatible memory)
        return False


class Stager:
    """Ring of ``nslots`` pinned slots of ``slot_bytes`` and ``threads`` host
    copy workers.  ``copy2d`` / ``copy`` enqueue jobs; ``flush`` issues every
    remaining DMA (all on ``stream``).  Not thread-safe: one user at a time
    (``stager()`` hands out one instance per device; its users --
    ``refine_and_fuse``, ``fuse``'s view upload, ``project_grid_overlay`` --
    hold the device's lock, ``fusion._device_lock``, while they use it).  Four copy threads by default
    (``DIVAS_STAGE_THREADS``): C3 pageable update 21-23 ms with 4, 24-25 with
    3 or 6, 27 with 8, 31-32 with 12 or 16 -- more threads contend for the
    host memory the DMAs read.  Slots of 8 MB x 12 measured best (16 MB x 16:
    24 ms, 4 MB x 24: 28 ms, 32 MB x 8: 28 ms)."""

    def __init__(self, slot_bytes=8 << 20, nslots=12, threads=4):
        import torch
        self.slot_bytes = int(slot_bytes)
        self.slots = [torch.empty(self.slot_bytes, dtype=torch.uint8, pin_memory=True)
                      for _ in range(nslots)]
        self.np_slots = [s.numpy() for s in self.slots]
        self.ptrs = [int(s.data_ptr()) for s in self.slots]
        self.events = [None] * nslots
        self.pool = cf.ThreadPoolExecutor(max_workers=threads)
        self.pending = collections.deque()
        self.next = 0
        self.stream = None
        self.bytes = 0

    def _issue_one(self):
        fut, slot, dst, dpitch, width, rows = self.pending.popleft()
        fut.result()
        _native.check(_native.lib().divas_copy2d_h2d(
            dst, dpitch, self.ptrs[slot], width, width, rows,
            _native.stream_handle(self.stream)), "divas_copy2d_h2d")
        import torch
        ev = torch.cuda.Event()
        ev.record(self.stream)
        self.events[slot] = ev

    def _chunk(self, dst, dpitch, src2d):
        """One slot's worth of whole rows of ``src2d`` (C-contiguous rows)."""
        rows, width = src2d.shape[0], src2d.shape[1] * src2d.itemsize
        slot = self.next
        self.next = (self.next + 1) % len(self.slots)
        # the slot's previous DMA must have finished before it is refilled;
        # meanwhile keep the copy engine fed with completed host copies
        while self.pending and self.pending[0][1] == slot:
            self._issue_one()
        if self.events[slot] is not None:
            self.events[slot].synchronize()
            self.events[slot] = None
        view = self.np_slots[slot][:rows * width].view(src2d.dtype).reshape(src2d.shape)
        fut = self.pool.submit(np.copyto, view, src2d)
        self.pending.append((fut, slot, dst, dpitch, width, rows))
        self.bytes += rows * width
        while self.pending and self.pending[0][0].done():
            self._issue_one()

    def copy2d(self, dst_ptr, dpitch, src2d, stream):
        """Rows of ``src2d`` (a 2-D numpy view, rows contiguous) to the device
        rectangle at ``dst_ptr`` with row pitch ``dpitch`` bytes."""
        self.stream = stream
        src2d = np.asarray(src2d)
        if src2d.ndim == 1:
            src2d = src2d.reshape(1, -1)
        width = src2d.shape[1] * src2d.itemsize
        if width > self.slot_bytes:                  # very wide rows: split columns
            step = self.slot_bytes // src2d.itemsize
            for c0 in range(0, src2d.shape[1], step):
                self.copy2d(dst_ptr + c0 * src2d.itemsize, dpitch, src2d[:, c0:c0 + step], stream)
            return
        per = max(1, self.slot_bytes // width)
        for r0 in range(0, src2d.shape[0], per):
            self._chunk(dst_ptr + r0 * dpitch, dpitch, src2d[r0:r0 + per])

    def copy(self, dst_ptr, src, stream):
        """A contiguous host array to contiguous device memory at ``dst_ptr``."""
        flat = np.ascontiguousarray(src).reshape(-1).view(np.uint8)
        n = flat.size
        row = self.slot_bytes
        full = n // row
        if full:
            self.copy2d(dst_ptr, row, flat[:full * row].reshape(full, row), stream)
        if n > full * row:
            self.copy2d(dst_ptr + full * row, row, flat[full * row:].reshape(1, -1), stream)

    def flush(self):
        """Issue every queued DMA (they complete asynchronously on the stream)."""
        while self.pending:
            self._issue_one()

    def discard(self):
        """Drop every queued job without issuing its DMA (after an error in
        the caller, whose device buffers may be released): wait for the host
        copies still running, so no slot is written afterwards."""
        while self.pending:
            fut = self.pending.popleft()[0]
            try:
                fut.result()
            except Exception:  # noqa: BLE001  (the caller's error is the one raised)
                pass


_STAGERS = {}
_LOCK = threading.Lock()


def stager(dev) -> Stager:
    key = str(dev)
    with _LOCK:
        if key not in _STAGERS:
            _STAGERS[key] = Stager(threads=int(os.environ.get("DIVAS_STAGE_THREADS", "4")))
        return _STAGERS[key]
