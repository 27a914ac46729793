"""HASF as a registered PyTorch operator (torch.library):

    from paper_1603_09337_b200 import register_torch_ops
    register_torch_ops()
    y = torch.ops.toposmooth_b200.hasf_batch(x_cuda_uint8_nhw, 5)          # (8,4) adjacency
    y = torch.ops.toposmooth_b200.hasf_batch(x, 4, 4, keep, avoid)           # (4,8), constraints

The CUDA implementation is smoothing.hasf_batch (the fused kernel through the C
ABI, smoothing.py:187-217 in the reference); the fake implementation gives the
output's shape and dtype for tracing.  There is no CPU implementation: the
operator fails on CPU tensors like every other compute entry of the package.
"""

from __future__ import annotations

_registered = False


def register_torch_ops() -> None:
    """Registers torch.ops.toposmooth_b200.hasf_batch once per process."""
    global _registered
    if _registered:
        return
    import torch

    from .grid import ADJ_48, ADJ_84
    from .smoothing import hasf_batch

    @torch.library.custom_op(
        "toposmooth_b200::hasf_batch", mutates_args=(), device_types="cuda",
        schema="(Tensor images, int r_max, int fg=8, Tensor? keep=None, Tensor? avoid=None) -> Tensor")
    def _hasf_batch(images, r_max, fg=8, keep=None, avoid=None):
        if fg not in (4, 8):
            raise ValueError(f"foreground adjacency must be 4 or 8, got {fg}")
        return hasf_batch(images, r_max, ADJ_84 if fg == 8 else ADJ_48, keep=keep, avoid=avoid)

    @_hasf_batch.register_fake
    def _(images, r_max, fg=8, keep=None, avoid=None):
        return torch.empty_like(images, dtype=torch.uint8)

    _registered = True
