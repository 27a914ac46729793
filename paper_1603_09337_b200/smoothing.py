"""Topology-preserving smoothing (HASF) on the B200 (mirrors smoothing.py:1-217).

`smooth`, `hasf`, `homotopic_cutting`, `homotopic_filling` keep the
reference's signatures, validation and error messages; the work runs in the
fused per-image kernel (csrc/ts_hasf.cu) through the C ABI.  `hasf_batch` is
the batched entry point (many independent images per launch) that fills the
GPU; it accepts numpy or torch (CUDA) [n, h, w] uint8/bool arrays.
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np

from . import _device as D
from ._lib import check, load
from .edt import SCHEDULERS
from .grid import ADJ_84, Adjacency, as_binary
from .morph import _check_radius


@dataclass(frozen=True)
class SmoothingConfig:
    """Filter order, constraint sets, adjacency, execution parameters (smoothing.py:31-40).
    `workers` / `scheduler` are validated for parity; the device schedule ignores them."""

    r_max: int
    adj: Adjacency = ADJ_84
    keep: np.ndarray | None = None
    avoid: np.ndarray | None = None
    workers: int = 1
    scheduler: str = "nps"


def _check_cfg(cfg: SmoothingConfig) -> None:
    """smoothing.py:43-48"""
    _check_radius(cfg.r_max)
    if cfg.workers < 1:
        raise ValueError("workers must be >= 1")
    if cfg.scheduler not in SCHEDULERS:
        raise ValueError(f"unknown scheduler {cfg.scheduler!r}")


def _run_single(fn_name, pix, *args, extra=None):
    import torch
    h, w = pix.shape
    d = D.to_device_u8(pix)[None]
    x = None if extra is None else D.to_device_u8(extra)[None]
    out = torch.empty_like(d)
    check(getattr(load(), fn_name)(d.data_ptr(), out.data_ptr(), 1, h, w, *args, D.ptr(x), D.stream_ptr()))
    return out[0].cpu().numpy()


def homotopic_cutting(img, keep, r, adj: Adjacency = ADJ_84, workers: int = 1, scheduler: str = "nps") -> np.ndarray:
    """Thin toward erode(img, r) | keep, then regrow inside dilate(thinned, r) & img
    (smoothing.py:149-165)."""
    pix = as_binary(img)
    keep = as_binary(keep)
    r = _check_radius(r)
    if keep.shape != pix.shape:
        raise ValueError(f"constraint shape {keep.shape} != image shape {pix.shape}")
    if np.any(keep & (pix ^ 1)):
        raise ValueError("keep-constraint pixels must be object pixels")
    return _run_single("ts_cutting_batch", pix, r, adj.fg, extra=keep)


def homotopic_filling(img, avoid, r, adj: Adjacency = ADJ_84, workers: int = 1, scheduler: str = "nps") -> np.ndarray:
    """Thicken inside dilate(img, r) minus avoid, then thin back toward
    erode(thickened, r) | img (smoothing.py:168-184)."""
    pix = as_binary(img)
    avoid = as_binary(avoid)
    r = _check_radius(r)
    if avoid.shape != pix.shape:
        raise ValueError(f"constraint shape {avoid.shape} != image shape {pix.shape}")
    if np.any(avoid & pix):
        raise ValueError("avoid-constraint pixels must be background pixels")
    return _run_single("ts_filling_batch", pix, r, adj.fg, extra=avoid)


def hasf(img, cfg: SmoothingConfig) -> np.ndarray:
    """Alternate cutting and filling at radii 1..r_max (smoothing.py:187-212)."""
    pix = as_binary(img)
    _check_cfg(cfg)
    keep = None if cfg.keep is None else as_binary(cfg.keep)
    avoid = None if cfg.avoid is None else as_binary(cfg.avoid)
    if (keep is not None and keep.shape != pix.shape) or (avoid is not None and avoid.shape != pix.shape):
        raise ValueError("constraint images must match the input shape")
    if keep is not None and avoid is not None and np.any(keep & avoid):
        raise ValueError("keep and avoid constraints overlap")
    if keep is not None and np.any(keep & (pix ^ 1)):
        raise ValueError("keep-constraint pixels must be object pixels")
    if avoid is not None and np.any(avoid & pix):
        raise ValueError("avoid-constraint pixels must be background pixels")
    import torch
    h, w = pix.shape
    d = D.to_device_u8(pix)[None]
    k = None if keep is None else D.to_device_u8(keep)[None]
    a = None if avoid is None else D.to_device_u8(avoid)[None]
    out = torch.empty_like(d)
    check(load().ts_hasf_batch(d.data_ptr(), out.data_ptr(), 1, h, w, int(cfg.r_max), cfg.adj.fg, D.ptr(k),
                               D.ptr(a), D.stream_ptr(), None))
    return out[0].cpu().numpy()


def smooth(img, r_max: int, workers: int = 1, scheduler: str = "nps") -> np.ndarray:
    """Unconstrained smoothing (smoothing.py:215-217)."""
    return hasf(img, SmoothingConfig(r_max=r_max, workers=workers, scheduler=scheduler))


class PendingCheck:
    """Device error flag of a non-blocking hasf_batch (ts_hasf_batch_async):
    check() waits for the flag (a 4-byte read in stream order) and raises the
    reference's exception classes like the blocking call."""

    def __init__(self, err):
        self.err = err

    def check(self) -> None:
        check(load().ts_check_device_error(int(self.err.item())))


def hasf_batch(images, r_max: int, adj: Adjacency = ADJ_84, keep=None, avoid=None, stats: bool = False,
               blocking: bool = True):
    """HASF on every image of an [n, h, w] batch in one launch.

    torch CUDA tensors stay on the device (returns a CUDA uint8 tensor); numpy
    input returns numpy.  Input/constraint validation happens on the device
    and raises ValueError with the reference's messages.  With stats=True also
    returns an int64 [n, 16] array: sweeps, fixpoint passes, engine calls, flips,
    cycles in prep / fixpoint passes / apply+re-examination / total, then
    tiny-sweep and dense-sweep breakdowns (see csrc/ts_internal.h kStatFields).
    With blocking=False (CUDA tensors only, no stats) nothing synchronizes:
    returns (out, PendingCheck); out is valid in stream order and
    PendingCheck.check() raises any device-side validation error.
    """
    import torch
    r_max = _check_radius(r_max)
    is_numpy = not isinstance(images, torch.Tensor)
    x = D.to_device_u8(images)
    if x.dim() != 3 or x.shape[1] < 1 or x.shape[2] < 1:
        raise ValueError(f"expected an [n, h, w] batch with positive dimensions, got shape {tuple(x.shape)}")
    n, h, w = x.shape
    k = None if keep is None else D.to_device_u8(keep)
    a = None if avoid is None else D.to_device_u8(avoid)
    for name, t in (("keep", k), ("avoid", a)):
        if t is not None and tuple(t.shape) != (n, h, w):
            raise ValueError(f"{name} constraint shape {tuple(t.shape)} != batch shape {(n, h, w)}")
    out = torch.empty_like(x)
    if not blocking:
        if is_numpy or stats:
            raise ValueError("blocking=False needs CUDA tensor input and stats=False")
        err = torch.zeros(1, dtype=torch.int32, device=x.device)
        check(load().ts_hasf_batch_async(x.data_ptr(), out.data_ptr(), n, h, w, r_max, adj.fg, D.ptr(k), D.ptr(a),
                                         D.stream_ptr(), err.data_ptr()))
        return out, PendingCheck(err)
    st = np.zeros((n, 36), np.int64) if stats else None
    check(load().ts_hasf_batch(x.data_ptr(), out.data_ptr(), n, h, w, r_max, adj.fg, D.ptr(k), D.ptr(a),
                               D.stream_ptr(), None if st is None else st.ctypes.data))
    res = out.cpu().numpy() if is_numpy else out
    return (res, st) if stats else res


def hasf_batch_host(images: np.ndarray, r_max: int, adj: Adjacency = ADJ_84, out: np.ndarray | None = None):
    """HASF on a host [n, h, w] uint8 batch through the C ABI's host-buffer entry
    (ts_hasf_batch_host: H2D copy, kernel, D2H copy inside the call)."""
    images = np.ascontiguousarray(images, dtype=np.uint8)
    if images.ndim != 3:
        raise ValueError("expected an [n, h, w] batch")
    n, h, w = images.shape
    if out is None:
        out = np.empty_like(images)
    D.require_cuda()
    check(load().ts_hasf_batch_host(images.ctypes.data, out.ctypes.data, n, h, w, _check_radius(r_max), adj.fg,
                                    None, None, D.stream_ptr()))
    return out
