"""Multi-GPU batching: one process per GPU, images sharded across ranks.

HASF images are independent units: each rank smooths a
contiguous shard of the batch with no data-path collective; the only
communication is an optional all-gather of the results and the
max-over-ranks timing reduce.  Uses torch.distributed (NCCL on GPUs, gloo in
the CPU tests).
"""

from __future__ import annotations

import numpy as np


def shard_range(n: int, rank: int, world: int) -> tuple[int, int]:
    """Balanced contiguous shard [start, stop) of n images for `rank`."""
    if world < 1 or not (0 <= rank < world):
        raise ValueError(f"bad rank {rank} for world size {world}")
    base, rem = divmod(int(n), world)
    start = rank * base + min(rank, rem)
    return start, start + base + (1 if rank < rem else 0)


def max_over_ranks(value: float, group=None) -> float:
    """Max of a per-rank scalar (e.g. device-timed milliseconds)."""
    import torch
    import torch.distributed as dist
    if not (dist.is_available() and dist.is_initialized()):
        return float(value)
    dev = "cuda" if dist.get_backend(group) == "nccl" else "cpu"
    t = torch.tensor([float(value)], dtype=torch.float64, device=dev)
    dist.all_reduce(t, op=dist.ReduceOp.MAX, group=group)
    return float(t.item())


def pack_rows(t):
    """uint8 {0,1} [k, h, w] tensor -> [k, h, ceil(w / 8)] bytes, MSB first
    (the P4 raster layout): the gather moves 1 bit per pixel."""
    import torch
    k, h, w = t.shape
    pad = (-w) % 8
    if pad:
        t = torch.nn.functional.pad(t, (0, pad))
    weights = (1 << torch.arange(7, -1, -1, device=t.device, dtype=torch.int32)).to(torch.uint8)
    return (t.view(k, h, -1, 8) * weights).sum(-1, dtype=torch.int32).to(torch.uint8)


def unpack_rows(p, w: int):
    import torch
    shifts = torch.arange(7, -1, -1, device=p.device, dtype=torch.uint8)
    bits = (p[..., None] >> shifts) & 1
    return bits.reshape(p.shape[0], p.shape[1], -1)[:, :, :w].contiguous()


def hasf_sharded(images, r_max: int, adj=None, group=None, fn=None) -> np.ndarray:
    """Smooth this rank's shard of a host [n, h, w] batch and all-gather the
    full [n, h, w] result on every rank.

    The gather moves bit-packed rows (1 bit per pixel, 8x fewer bytes than
    uint8); with NCCL the shard stays on the rank's GPU from the kernel to the
    collective.  `fn(shard, r_max, adj)` defaults to the device path
    (smoothing.hasf_batch); tests substitute the CPU oracle to exercise the
    collective logic without a GPU.
    """
    import torch
    import torch.distributed as dist

    from .grid import ADJ_84
    adj = ADJ_84 if adj is None else adj
    images = np.ascontiguousarray(images, dtype=np.uint8)
    n, h, w = images.shape
    world = dist.get_world_size(group) if dist.is_initialized() else 1
    rank = dist.get_rank(group) if dist.is_initialized() else 0
    if fn is None:
        from .smoothing import hasf_batch
        fn = hasf_batch
    s0, s1 = shard_range(n, rank, world)
    grouped = dist.is_initialized()   # a process group exists (also a single-rank one): gather through it
    dev = "cuda" if grouped and dist.get_backend(group) == "nccl" else "cpu"
    shard = images[s0:s1]
    mine = fn(torch.from_numpy(shard).to(dev) if dev == "cuda" else shard, r_max, adj)
    mine = mine if isinstance(mine, torch.Tensor) else torch.from_numpy(np.asarray(mine, dtype=np.uint8))
    if not grouped:
        return mine.cpu().numpy()
    chunk = -(-n // world)   # ceil: equal-size padded chunks for all_gather
    buf = torch.zeros((chunk, h, (w + 7) // 8), dtype=torch.uint8, device=dev)
    if s1 > s0:
        buf[: s1 - s0] = pack_rows(mine.to(dev))
    parts = [torch.empty_like(buf) for _ in range(world)]
    dist.all_gather(parts, buf, group=group)
    out = np.empty((n, h, w), np.uint8)
    for r in range(world):
        a, b = shard_range(n, r, world)
        if b > a:
            out[a:b] = unpack_rows(parts[r][: b - a], w).cpu().numpy()
    return out
