"""Device plumbing: torch for CUDA memory and streams (not for compute)."""

from __future__ import annotations

import numpy as np
import torch


def require_cuda() -> torch.device:
    if not torch.cuda.is_available():
        raise RuntimeError("toposmooth_b200 needs a CUDA device (no CPU fallback)")
    return torch.device("cuda", torch.cuda.current_device())


def stream_ptr() -> int:
    return torch.cuda.current_stream().cuda_stream


def ptr(t) -> int | None:
    return None if t is None else t.data_ptr()


def to_device_u8(a) -> torch.Tensor:
    """Contiguous uint8 CUDA tensor (bool -> uint8) from numpy or torch."""
    dev = require_cuda()
    if isinstance(a, torch.Tensor):
        t = a
        if t.dtype == torch.bool:
            t = t.to(torch.uint8)
        if t.dtype != torch.uint8:
            t = t.to(torch.uint8)
        return t.to(dev).contiguous()
    return torch.from_numpy(np.ascontiguousarray(a, dtype=np.uint8)).to(dev)


def to_device_i64(a) -> torch.Tensor:
    dev = require_cuda()
    if isinstance(a, torch.Tensor):
        return a.to(dev, torch.int64).contiguous()
    return torch.from_numpy(np.ascontiguousarray(a, dtype=np.int64)).to(dev)
