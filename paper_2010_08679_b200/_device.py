"""Device-side plumbing shared by the host mirror: uploads, flags, sync checks.

Scratch buffers come from torch's caching allocator per call, so concurrent
callers (the reference's shard pool threads, engine.py:357-372) never share
mutable state.
"""

from __future__ import annotations

import numpy as np
import torch

from . import _lib


def device_of(dev=None) -> torch.device:
    _lib.require_cuda()
    if dev is None:
        return torch.device("cuda", torch.cuda.current_device())
    dev = torch.device(dev)
    if dev.type != "cuda":
        raise ValueError(f"paper_2010_08679_b200 runs on CUDA devices only, got {dev}")
    cur = torch.cuda.current_device()
    if dev.index is None:
        dev = torch.device("cuda", cur)
    elif dev.index != cur:
        # the entry points launch on the current device's stream (and the C
        # side caches per-device properties of cudaGetDevice): refuse a launch
        # that would pair another device's pointers with this device
        raise ValueError(f"paper_2010_08679_b200: {dev} is not the current device cuda:{cur}; "
                         "call torch.cuda.set_device() or run under torch.cuda.device()")
    return dev


def is_torch(x) -> bool:
    return isinstance(x, torch.Tensor)


def to_device(x, dtype: torch.dtype, device: torch.device) -> torch.Tensor:
    """Contiguous device tensor of `dtype` (zero-copy for matching CUDA tensors)."""
    if isinstance(x, torch.Tensor):
        t = x
        if t.device != device:
            t = t.to(device, non_blocking=True)
        if t.dtype != dtype:
            t = t.to(dtype)
        return t.contiguous()
    a = np.ascontiguousarray(x, dtype=torch_to_numpy(dtype))
    if not a.flags.writeable:  # torch.from_numpy warns on read-only views
        a = a.copy()
    return torch.from_numpy(a).to(device, non_blocking=False)


def torch_to_numpy(dtype: torch.dtype):
    return {
        torch.float32: np.float32,
        torch.float64: np.float64,
        torch.int64: np.int64,
        torch.int32: np.int32,
        torch.uint8: np.uint8,
    }[dtype]


def new_flags(device: torch.device) -> torch.Tensor:
    return torch.zeros(1, dtype=torch.int32, device=device)


def check_flags(flags: torch.Tensor, what: str) -> None:
    """Synchronise on the flag word and raise the reference exception."""
    v = int(flags.item()) & 0xFFFFFFFF
    _lib.raise_flags(v, what)


def like_input(out: torch.Tensor, ref):
    """Return numpy when the caller passed host arrays (reference types)."""
    if isinstance(ref, torch.Tensor):
        return out
    return out.cpu().numpy()
