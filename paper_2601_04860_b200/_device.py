"""Device plumbing: numpy <-> CUDA tensors (PyTorch is the allocator / stream
provider only; all arithmetic on the path runs in libdivas_b200.so)."""

from __future__ import annotations

import numpy as np

_NP2TORCH = None


def _dtype(np_dtype):
    global _NP2TORCH
    import torch
    if _NP2TORCH is None:
        _NP2TORCH = {np.dtype(np.float32): torch.float32, np.dtype(np.float64): torch.float64,
                     np.dtype(np.int32): torch.int32, np.dtype(np.int64): torch.int64,
                     np.dtype(np.uint8): torch.uint8, np.dtype(np.bool_): torch.bool}
    return _NP2TORCH[np.dtype(np_dtype)]


def device():
    """The current CUDA device; raises when there is none (no CPU fallback)."""
    import torch
    if not torch.cuda.is_available():
        raise RuntimeError("paper_2601_04860_b200 needs a CUDA device (B200, sm_100a); "
                           "there is no CPU fallback")
    return torch.device("cuda", torch.cuda.current_device())


def as_device(a, np_dtype, dev, non_blocking=False):
    """Contiguous CUDA tensor of dtype ``np_dtype`` holding ``a`` (numpy or torch)."""
    import torch
    if isinstance(a, torch.Tensor):
        t = a.to(device=dev, dtype=_dtype(np_dtype), non_blocking=non_blocking)
        return t.contiguous()
    arr = np.ascontiguousarray(a, dtype=np_dtype)
    return torch.from_numpy(arr).to(dev, non_blocking=non_blocking)


def empty(shape, np_dtype, dev):
    import torch
    return torch.empty(tuple(shape), dtype=_dtype(np_dtype), device=dev)


def zeros(shape, np_dtype, dev):
    import torch
    return torch.zeros(tuple(shape), dtype=_dtype(np_dtype), device=dev)
