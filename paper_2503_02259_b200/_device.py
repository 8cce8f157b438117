"""Device plumbing: torch owns HBM allocations and streams; libkgp does the compute.

There is no CPU path. Every helper raises ``KernelGpError`` when no CUDA device
is visible, so a product call can never silently run on the host.
"""

from __future__ import annotations

import numpy as np

from paper_2503_02259_b200.errors import KernelGpError

_torch = None


def torch():
    global _torch
    if _torch is None:
        import torch as _t

        _torch = _t
    return _torch


def device():
    t = torch()
    if not t.cuda.is_available():
        raise KernelGpError("no CUDA device visible: paper_2503_02259_b200 runs only on the GPU "
                            "(there is no CPU fallback)")
    return t.device("cuda", t.cuda.current_device())


def stream_ptr() -> int:
    device()
    return torch().cuda.current_stream().cuda_stream


def is_tensor(x) -> bool:
    t = torch()
    return isinstance(x, t.Tensor)


def to_device(a, dtype=None):
    """Host array-like -> contiguous fp64 CUDA tensor (torch tensors pass through)."""
    t = torch()
    dev = device()
    if isinstance(a, t.Tensor):
        return a.to(device=dev, dtype=dtype or t.float64).contiguous()
    arr = np.ascontiguousarray(a, dtype=np.float64 if dtype is None else None)
    if not arr.flags.writeable:  # e.g. the engine's read-only X copy; torch wants writable memory
        arr = arr.copy()
    return t.from_numpy(arr).to(dev, non_blocking=False)


def to_host(x) -> np.ndarray:
    return x.detach().cpu().numpy()


def empty(shape, dtype=None):
    t = torch()
    return t.empty(shape, dtype=dtype or t.float64, device=device())


def zeros(shape, dtype=None):
    t = torch()
    return t.zeros(shape, dtype=dtype or t.float64, device=device())
