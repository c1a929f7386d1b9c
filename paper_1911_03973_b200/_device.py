"""Device plumbing: torch tensors in, raw pointers and the current stream out."""

from __future__ import annotations

import ctypes

import numpy as np
import torch


def device() -> torch.device:
    """The CUDA device every tensor of this package lives on (no CPU fallback)."""
    if not torch.cuda.is_available():
        raise RuntimeError(
            "paper_1911_03973_b200 computes on a CUDA device (B200, sm_100a); "
            "none is visible and there is no CPU fallback")
    return torch.device("cuda", torch.cuda.current_device())


def stream() -> ctypes.c_void_p:
    return ctypes.c_void_p(torch.cuda.current_stream().cuda_stream)


def ptr(t) -> ctypes.c_void_p:
    if t is None:
        return ctypes.c_void_p(0)
    return ctypes.c_void_p(t.data_ptr())


def to_device(x, dtype, contiguous=True) -> torch.Tensor:
    """numpy / torch (any device) -> contiguous tensor of `dtype` on the device."""
    dev = device()
    if isinstance(x, torch.Tensor):
        t = x
    else:
        a = np.ascontiguousarray(np.asarray(x))
        if not a.flags.writeable:  # torch.from_numpy needs a writable buffer
            a = a.copy()
        t = torch.from_numpy(a)
    if t.device != dev or t.dtype != dtype:
        pinned = t.device.type == "cpu" and t.is_pinned()
        t = t.to(device=dev, dtype=dtype, non_blocking=pinned)
    if contiguous and not t.is_contiguous():
        t = t.contiguous()
    return t


def f64(x) -> torch.Tensor:
    return to_device(x, torch.float64)


def i64(x) -> torch.Tensor:
    return to_device(x, torch.int64)


def i32(x) -> torch.Tensor:
    return to_device(x, torch.int32)


def empty(shape, dtype=torch.float64) -> torch.Tensor:
    return torch.empty(shape, dtype=dtype, device=device())


def zeros(shape, dtype=torch.float64) -> torch.Tensor:
    return torch.zeros(shape, dtype=dtype, device=device())
