"""Exact squared Euclidean distance transform on the device (mirrors edt.py:1-211).

edt_squared / edt_phase1_columns / edt_phase2_rows run the K1 kernels of
csrc/ts_edt.cu (column sweeps, then per-row lower envelopes, int64 output
with the INF = h^2 + w^2 + 1 sentinel).  `workers`/`scheduler` are accepted
and validated for API parity; on the GPU they do not change the schedule.
"""

from __future__ import annotations

import numpy as np

from . import _device as D
from ._lib import check, load
from .grid import as_binary

SCHEDULERS = ("nps", "strided", "system")   # sched.py:22


def _check_exec(workers, scheduler):
    if workers < 1:
        raise ValueError("workers must be >= 1")
    if scheduler not in SCHEDULERS:
        raise ValueError(f"unknown scheduler {scheduler!r}")


def inf_value(shape) -> int:
    """edt.py:25-28"""
    h, w = shape
    return int(h) * int(h) + int(w) * int(w) + 1


def sep(i: int, u: int, g_i: int, g_u: int) -> int:
    """edt.py:31-42 (scalar host arithmetic, floor division)."""
    if i >= u:
        raise ValueError(f"sep requires i < u, got i={i}, u={u}")
    if g_i < 0 or g_u < 0:
        raise ValueError("column distances must be non-negative")
    return (u * u - i * i + g_u * g_u - g_i * g_i) // (2 * (u - i))


def _edt_device(pix_dev, mode: int):
    """[n,h,w] uint8 CUDA tensor -> int64 CUDA tensor (mode 0: to objects,
    mode 1: to background incl. window exterior)."""
    import torch
    n, h, w = pix_dev.shape
    out = torch.empty((n, h, w), dtype=torch.int64, device=pix_dev.device)
    check(load().ts_edt_sq_batch(pix_dev.data_ptr(), out.data_ptr(), n, h, w, mode, D.stream_ptr()))
    return out


def edt_squared(img, workers: int = 1, scheduler: str = "nps") -> np.ndarray:
    """Exact squared distance to the nearest object pixel (edt.py:173-187)."""
    pix = as_binary(img)
    _check_exec(workers, scheduler)
    return _edt_device(D.to_device_u8(pix)[None], 0)[0].cpu().numpy()


def _check_assignment(assignment, count):
    if assignment is None:
        return
    seen = np.zeros(count, dtype=bool)
    total = 0
    for bucket in assignment.buckets:
        for i in np.asarray(bucket, dtype=np.int64):
            if i < 0 or i >= count:
                raise ValueError(f"task index {i} outside 0..{count - 1}")
            if seen[i]:
                raise ValueError(f"task index {i} assigned more than once")
            seen[i] = True
            total += 1
    if total != count:
        raise ValueError(f"assignment covers {total} of {count} tasks")


def edt_phase1_columns(img, assignment=None) -> np.ndarray:
    """Vertical distances G (edt.py:122-136); any exact column assignment gives
    the same grid, so it is only validated."""
    import torch
    pix = as_binary(img)
    h, w = pix.shape
    _check_assignment(assignment, w)
    d = D.to_device_u8(pix)
    g = torch.empty((1, h, w), dtype=torch.int64, device=d.device)
    check(load().ts_edt_phase1_batch(d.data_ptr(), g.data_ptr(), 1, h, w, D.stream_ptr()))
    return g[0].cpu().numpy()


def edt_phase2_rows(g, assignment=None) -> np.ndarray:
    """Squared distances from the column-distance grid (edt.py:139-149)."""
    import torch
    g = np.ascontiguousarray(g, dtype=np.int64)
    if g.ndim != 2:
        raise ValueError("column-distance grid must be 2D")
    h, w = g.shape
    _check_assignment(assignment, h)
    gd = D.to_device_i64(g)
    out = torch.empty((1, h, w), dtype=torch.int64, device=gd.device)
    check(load().ts_edt_phase2_batch(gd.data_ptr(), out.data_ptr(), 1, h, w, D.stream_ptr()))
    return out[0].cpu().numpy()


def edt_bruteforce(img) -> np.ndarray:
    """Definitional O(n^2 m^2) transform (edt.py:190-211), host-side test helper."""
    pix = as_binary(img)
    h, w = pix.shape
    inf = inf_value(pix.shape)
    rows, cols = np.nonzero(pix)
    best = np.full((h, w), inf, dtype=np.int64)
    if rows.size == 0:
        return best
    rr = np.arange(h, dtype=np.int64)[:, None]
    cc = np.arange(w, dtype=np.int64)[None, :]
    for start in range(0, rows.size, 128):
        br = rows[start:start + 128].astype(np.int64)[:, None, None]
        bc = cols[start:start + 128].astype(np.int64)[:, None, None]
        d = (rr[None, :, :] - br) ** 2 + (cc[None, :, :] - bc) ** 2
        np.minimum(best, d.min(axis=0), out=best)
    return best
