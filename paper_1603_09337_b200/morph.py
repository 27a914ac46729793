"""Ball dilation / erosion by thresholding the device EDT (mirrors morph.py:1-59)."""

from __future__ import annotations

import numpy as np

from . import _device as D
from ._lib import check, load
from .edt import _check_exec, _edt_device
from .grid import as_binary


def _check_radius(r) -> int:
    """morph.py:18-22"""
    r = int(r)
    if r < 0:
        raise ValueError("ball radius must be >= 0")
    return r


def background_distances(img, workers: int = 1, scheduler: str = "nps") -> np.ndarray:
    """Squared distance to the nearest background pixel, window exterior
    included (morph.py:34-42)."""
    pix = as_binary(img)
    _check_exec(workers, scheduler)
    return _edt_device(D.to_device_u8(pix)[None], 1)[0].cpu().numpy()


def _threshold(img, r, fn_name):
    import torch
    pix = as_binary(img)
    d = D.to_device_u8(pix)[None]
    out = torch.empty_like(d)
    check(getattr(load(), fn_name)(d.data_ptr(), out.data_ptr(), 1, pix.shape[0], pix.shape[1], r, D.stream_ptr()))
    return out[0].cpu().numpy()


def dilate(img, r, workers: int = 1, scheduler: str = "nps") -> np.ndarray:
    """Union of Euclidean discs of radius r (morph.py:45-49)."""
    r = _check_radius(r)
    _check_exec(workers, scheduler)
    return _threshold(img, r, "ts_dilate_batch")


def erode(img, r, workers: int = 1, scheduler: str = "nps") -> np.ndarray:
    """Pixels whose radius-r disc lies inside the object (morph.py:52-59)."""
    r = _check_radius(r)
    _check_exec(workers, scheduler)
    return _threshold(img, r, "ts_erode_batch")
