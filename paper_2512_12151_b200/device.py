"""Device buffers: torch CUDA tensors used purely as FP64 storage."""

from __future__ import annotations

import numpy as np

_torch = None


def torch():
    global _torch
    if _torch is None:
        import torch as t
        _torch = t
    return _torch


def require_cuda():
    t = torch()
    if not t.cuda.is_available():
        raise RuntimeError("paper_2512_12151_b200 needs a CUDA device (B200, sm_100a); there is no CPU path")
    return t


def to_dev(a, dtype=None):
    """numpy -> contiguous CUDA tensor (float64 unless dtype given)."""
    t = require_cuda()
    arr = np.ascontiguousarray(a, dtype=dtype or np.float64)
    return t.from_numpy(arr).to("cuda", non_blocking=False)


def empty(shape, dtype=None):
    t = require_cuda()
    return t.empty(shape, dtype=dtype or t.float64, device="cuda")


def zeros(shape, dtype=None):
    t = require_cuda()
    return t.zeros(shape, dtype=dtype or t.float64, device="cuda")


def to_host(x):
    return x.detach().to("cpu").numpy()
