"""Local topology and the priority-ordered homotopic thinning / thickening
engine on the device (mirrors topo.py:1-354).

The connectivity tables come from the native library (restated from their
definition, topo.py:44-84).  neighborhood_codes / simple_point_mask run the
classifier kernel (LUT staged in shared memory); homotopic_thin /
homotopic_thicken run the fused kernel's engine (csrc/ts_hasf.cu) with
arbitrary int64 priorities, reproducing the reference's removal order
exactly, including max_iter (number of sweeps).
"""

from __future__ import annotations

import ctypes
from typing import NamedTuple

import numpy as np

from . import _device as D
from ._lib import check, load
from .edt import _check_exec
from .grid import ADJ_84, Adjacency, as_binary

_OFFSETS = ((-1, -1), (-1, 0), (-1, 1), (0, -1), (0, 1), (1, -1), (1, 0), (1, 1))   # topo.py:35


def _comp_count(mask: int, conn: int) -> int:
    """Components of the set neighbours of a 3x3 window's centre (conn-adjacent
    to each other) that touch the centre under conn (topo.py:44-76)."""
    parent = list(range(8))

    def find(a):
        while parent[a] != a:
            parent[a] = parent[parent[a]]
            a = parent[a]
        return a

    for a in range(8):
        for b in range(a + 1, 8):
            if not ((mask >> a) & 1 and (mask >> b) & 1):
                continue
            dr = abs(_OFFSETS[a][0] - _OFFSETS[b][0])
            dc = abs(_OFFSETS[a][1] - _OFFSETS[b][1])
            if (dr + dc == 1) if conn == 4 else (dr <= 1 and dc <= 1):
                parent[find(a)] = find(b)
    roots = {find(a) for a in range(8)
             if (mask >> a) & 1 and (conn == 8 or _OFFSETS[a][0] == 0 or _OFFSETS[a][1] == 0)}
    return len(roots)


def _tables():
    """T8/T4 and the simple-point LUTs (topo.py:79-84), built at import on the
    host -- no native library load, so importing the package (e.g. for its
    workload generators) never maps libtoposmooth_b200.so.  The library holds
    the same tables (ts_connectivity_tables; tests check they agree)."""
    t8 = np.array([_comp_count(m, 8) for m in range(256)], np.uint8)
    t4 = np.array([_comp_count(m, 4) for m in range(256)], np.uint8)
    inv = np.arange(256) ^ 0xFF
    s84 = ((t8 == 1) & (t4[inv] == 1)).astype(np.uint8)
    s48 = ((t4 == 1) & (t8[inv] == 1)).astype(np.uint8)
    return t8, t4, s84, s48


def native_tables():
    """The library's copy of the four tables (ts_connectivity_tables)."""
    bufs = [(ctypes.c_uint8 * 256)() for _ in range(4)]
    check(load().ts_connectivity_tables(*[ctypes.addressof(b) for b in bufs]))
    return [np.frombuffer(b, dtype=np.uint8).copy() for b in bufs]


T8_TABLE, T4_TABLE, SIMPLE_84, SIMPLE_48 = _tables()


def _simple_lut(adj: Adjacency) -> np.ndarray:
    return SIMPLE_84 if adj.fg == 8 else SIMPLE_48


class TopoClassification(NamedTuple):
    fg_components: int
    bg_components: int
    simple: bool


def _code_at(pix, r, c) -> int:
    h, w = pix.shape
    code = 0
    for k, (dr, dc) in enumerate(_OFFSETS):
        nr, nc = r + dr, c + dc
        if 0 <= nr < h and 0 <= nc < w and pix[nr, nc]:
            code |= 1 << k
    return code


def connectivity_numbers(img, p, adj: Adjacency = ADJ_84) -> TopoClassification:
    """Connectivity numbers of p's punctured 3x3 neighbourhood (topo.py:119-136)."""
    pix = as_binary(img)
    r, c = p
    h, w = pix.shape
    if not (0 <= r < h and 0 <= c < w):
        raise ValueError(f"point {p!r} outside {h}x{w} image")
    code = _code_at(pix, r, c)
    if adj.fg == 8:
        t, tbar = int(T8_TABLE[code]), int(T4_TABLE[code ^ 0xFF])
    else:
        t, tbar = int(T4_TABLE[code]), int(T8_TABLE[code ^ 0xFF])
    return TopoClassification(t, tbar, t == 1 and tbar == 1)


def is_simple(img, p, adj: Adjacency = ADJ_84) -> bool:
    """topo.py:139-141"""
    return connectivity_numbers(img, p, adj).simple


def neighborhood_codes(img) -> np.ndarray:
    """Per-pixel 8-bit mask of object neighbours (topo.py:97-106), on the device."""
    import torch
    pix = as_binary(img)
    d = D.to_device_u8(pix)[None]
    out = torch.empty_like(d)
    check(load().ts_neighborhood_codes_batch(d.data_ptr(), out.data_ptr(), 1, pix.shape[0], pix.shape[1],
                                             D.stream_ptr()))
    return out[0].cpu().numpy()


def simple_point_mask(img, adj: Adjacency = ADJ_84) -> np.ndarray:
    """Boolean mask of simple object pixels (topo.py:144-148), on the device."""
    import torch
    pix = as_binary(img)
    d = D.to_device_u8(pix)[None]
    out = torch.empty_like(d)
    check(load().ts_simple_point_mask_batch(d.data_ptr(), out.data_ptr(), 1, pix.shape[0], pix.shape[1], adj.fg,
                                            D.stream_ptr()))
    return out[0].cpu().numpy().astype(bool)


def _check_priority(priority, shape, key_space):
    priority = np.ascontiguousarray(priority, dtype=np.int64)
    if priority.shape != shape:
        raise ValueError(f"priority shape {priority.shape} != image shape {shape}")
    if priority.size:
        lo, hi = int(priority.min()), int(priority.max())
        if lo < 0 or hi >= (1 << 62) // key_space:
            raise ValueError("priority values must be non-negative and fit the packed queue key")
    return priority


def _check_thin_args(img, keep, priority):
    """topo.py:261-276"""
    pix = as_binary(img)
    keep = as_binary(keep)
    if keep.shape != pix.shape:
        raise ValueError(f"constraint shape {keep.shape} != image shape {pix.shape}")
    if np.any(keep & (pix ^ 1)):
        raise ValueError("constraint pixels must be a subset of the object pixels")
    priority = _check_priority(priority, pix.shape, priority_size(pix.shape))
    return pix, keep, priority


def priority_size(shape):
    return int(np.prod(shape))


def _engine(fn_name, pix, mask, priority, adj, max_iter):
    import torch
    h, w = pix.shape
    d = D.to_device_u8(pix)[None]
    m = D.to_device_u8(mask)[None]
    pr = D.to_device_i64(priority)[None]
    out = torch.empty_like(d)
    # topo.py:298: a negative bound, like None, means "run to stability"
    mi = -1 if max_iter is None else max(-1, int(max_iter))
    check(getattr(load(), fn_name)(d.data_ptr(), m.data_ptr(), pr.data_ptr(), out.data_ptr(), 1, h, w, adj.fg, mi,
                                   D.stream_ptr()))
    return out[0].cpu().numpy()


def homotopic_thin(img, keep, priority, adj: Adjacency = ADJ_84, max_iter: int | None = None,
                   workers: int = 1, scheduler: str = "nps") -> np.ndarray:
    """Remove simple points outside `keep`, lowest (priority, raster index)
    first, to stability or max_iter sweeps (topo.py:303-314)."""
    pix, keep, priority = _check_thin_args(img, keep, priority)
    _check_exec(workers, scheduler)
    return _engine("ts_thin_batch", pix, keep, priority, adj, max_iter)


def homotopic_thicken(img, allowed, priority, adj: Adjacency = ADJ_84, max_iter: int | None = None,
                      workers: int = 1, scheduler: str = "nps") -> np.ndarray:
    """Add points simple for the background inside `allowed` (topo.py:317-342);
    equal to thinning the ring-padded complement under adj.dual()."""
    pix = as_binary(img)
    allowed = as_binary(allowed)
    if allowed.shape != pix.shape:
        raise ValueError(f"constraint shape {allowed.shape} != image shape {pix.shape}")
    if np.any(pix & (allowed ^ 1)):
        raise ValueError("object pixels must be a subset of the allowed set")
    priority = _check_priority(priority, pix.shape, (pix.shape[0] + 2) * (pix.shape[1] + 2))
    _check_exec(workers, scheduler)
    return _engine("ts_thicken_batch", pix, allowed, priority, adj, max_iter)
