"""Host/device array plumbing for the operator API (torch is the allocator)."""

from __future__ import annotations

import numpy as np


def is_torch(a) -> bool:
    return type(a).__module__.startswith("torch")


def require_cuda():
    import torch
    if not torch.cuda.is_available():
        raise RuntimeError("paper_2605_10729_b200 needs a CUDA device (B200); "
                           "there is no CPU implementation of the PIF step")
    return torch


def default_device(like=None):
    torch = require_cuda()
    if like is not None and is_torch(like) and like.is_cuda:
        return like.device
    return torch.device("cuda", torch.cuda.current_device())


def as_device(a, *, complex_: bool = False, device=None, contiguous: bool = True):
    """numpy / torch -> float64 (or complex128) CUDA tensor."""
    torch = require_cuda()
    dev = device if device is not None else default_device(a)
    dt = torch.complex128 if complex_ else torch.float64
    if is_torch(a):
        t = a.to(device=dev, dtype=dt)
    else:
        arr = np.asarray(a)
        arr = arr.astype(np.complex128 if complex_ else np.float64, copy=False)
        t = torch.from_numpy(np.ascontiguousarray(arr)).to(dev)
    return t.contiguous() if contiguous else t


def like_input(t, src):
    """Return t as numpy if src was numpy, else as the torch tensor."""
    if is_torch(src):
        return t
    return t.detach().cpu().numpy()
