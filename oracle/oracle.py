"""ctypes front end of the C oracle (hasf_oracle.c) -- TEST INFRASTRUCTURE ONLY.

Each function names the reference function it restates
(/root/reference/pkg/src/toposmooth/<file>:<lines>).  Inputs are assumed valid
(the reference's validation is mirrored by the product package, not here).
"""

from __future__ import annotations

import ctypes
import os
import subprocess
import threading

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_LIB_PATH = os.path.join(_HERE, "liboracle.so")
_lib = None
_lock = threading.Lock()

_u8p = ctypes.POINTER(ctypes.c_uint8)
_i64p = ctypes.POINTER(ctypes.c_int64)


def build() -> str:
    """Compile liboracle.so with gcc (oracle/Makefile)."""
    subprocess.run(["make", "-s", "-C", _HERE], check=True)
    return _LIB_PATH


def _load():
    global _lib
    with _lock:
        if _lib is not None:
            return _lib
        src = os.path.join(_HERE, "hasf_oracle.c")
        if not os.path.exists(_LIB_PATH) or os.path.getmtime(_LIB_PATH) < os.path.getmtime(src):
            build()
        lib = ctypes.CDLL(_LIB_PATH)
        i, i64 = ctypes.c_int, ctypes.c_int64
        sigs = {
            "orc_sep": ([i64, i64, i64, i64], i64),
            "orc_edt": ([_u8p, _i64p, i, i, i], None),
            "orc_edt_phase1": ([_u8p, _i64p, i, i], None),
            "orc_edt_phase2": ([_i64p, _i64p, i, i], None),
            "orc_luts": ([_u8p, _u8p, _u8p, _u8p], None),
            "orc_homotopic_thin": ([_u8p, _u8p, _i64p, i, i64, _u8p, i, i], i64),
            "orc_homotopic_thicken": ([_u8p, _u8p, _i64p, i, i64, _u8p, i, i], i64),
            "orc_cutting": ([_u8p, _u8p, i, i, _u8p, i, i], None),
            "orc_filling": ([_u8p, _u8p, i, i, _u8p, i, i], None),
            "orc_hasf": ([_u8p, _u8p, _u8p, i, i, _u8p, i, i], None),
            "orc_hasf_batch": ([_u8p, _u8p, _u8p, i64, i, i, i, i, _u8p, i], None),
        }
        for name, (argt, rest) in sigs.items():
            fn = getattr(lib, name)
            fn.argtypes = argt
            fn.restype = rest
        _lib = lib
        return lib


def _u8(a):
    a = np.ascontiguousarray(a, dtype=np.uint8)
    return a, a.ctypes.data_as(_u8p)


def _i64(a):
    a = np.ascontiguousarray(a, dtype=np.int64)
    return a, a.ctypes.data_as(_i64p)


def inf_value(shape) -> int:
    """edt.py:25-28"""
    h, w = shape
    return int(h) * int(h) + int(w) * int(w) + 1


def sep(i, u, g_i, g_u) -> int:
    """edt.py:31-42 (floor division)."""
    return int(_load().orc_sep(i, u, g_i, g_u))


def edt_squared(img, invert: bool = False) -> np.ndarray:
    """edt.py:152-187 (both phases; invert=True measures distance to background)."""
    pix, pp = _u8(img)
    h, w = pix.shape
    out = np.empty((h, w), np.int64)
    _load().orc_edt(pp, out.ctypes.data_as(_i64p), h, w, int(bool(invert)))
    return out


def edt_phase1_columns(img) -> np.ndarray:
    """edt.py:45-71, 122-136"""
    pix, pp = _u8(img)
    h, w = pix.shape
    g = np.empty((h, w), np.int64)
    _load().orc_edt_phase1(pp, g.ctypes.data_as(_i64p), h, w)
    return g


def edt_phase2_rows(g) -> np.ndarray:
    """edt.py:74-119, 139-149"""
    g, gp = _i64(g)
    h, w = g.shape
    out = np.empty((h, w), np.int64)
    _load().orc_edt_phase2(gp, out.ctypes.data_as(_i64p), h, w)
    return out


def border_distances_sq(shape) -> np.ndarray:
    """morph.py:25-31"""
    h, w = shape
    i = np.arange(h, dtype=np.int64)[:, None]
    j = np.arange(w, dtype=np.int64)[None, :]
    ring = np.minimum(np.minimum(i + 1, h - i), np.minimum(j + 1, w - j))
    return ring * ring


def background_distances(img) -> np.ndarray:
    """morph.py:34-42"""
    pix = np.ascontiguousarray(img, np.uint8)
    return np.minimum(edt_squared(pix ^ 1), border_distances_sq(pix.shape))


def dilate(img, r) -> np.ndarray:
    """morph.py:45-49"""
    return (edt_squared(img) <= int(r) * int(r)).astype(np.uint8)


def erode(img, r) -> np.ndarray:
    """morph.py:52-59"""
    return (background_distances(img) > int(r) * int(r)).astype(np.uint8)


def luts():
    """topo.py:44-84: (T8, T4, SIMPLE_84, SIMPLE_48) as uint8[256]."""
    t8, t4, s84, s48 = (np.empty(256, np.uint8) for _ in range(4))
    _load().orc_luts(*(a.ctypes.data_as(_u8p) for a in (t8, t4, s84, s48)))
    return t8, t4, s84, s48


_OFFSETS = ((-1, -1), (-1, 0), (-1, 1), (0, -1), (0, 1), (1, -1), (1, 0), (1, 1))


def neighborhood_codes(img) -> np.ndarray:
    """topo.py:97-106"""
    pix = np.ascontiguousarray(img, np.uint8)
    h, w = pix.shape
    padded = np.zeros((h + 2, w + 2), np.uint8)
    padded[1:-1, 1:-1] = pix
    code = np.zeros((h, w), np.uint8)
    for k, (dr, dc) in enumerate(_OFFSETS):
        code |= padded[1 + dr:1 + dr + h, 1 + dc:1 + dc + w] << np.uint8(k)
    return code


def simple_point_mask(img, fg: int = 8) -> np.ndarray:
    """topo.py:144-148"""
    pix = np.ascontiguousarray(img, np.uint8)
    lut = luts()[2 if fg == 8 else 3]
    return (pix == 1) & (lut[neighborhood_codes(pix)] == 1)


def homotopic_thin(img, keep, priority, fg: int = 8, max_iter=None):
    """topo.py:279-314 (heap engine topo.py:211-258)."""
    pix, pp = _u8(img)
    keep, kp = _u8(keep)
    prio, prp = _i64(priority)
    out = np.empty_like(pix)
    _load().orc_homotopic_thin(pp, kp, prp, fg, -1 if max_iter is None else int(max_iter),
                               out.ctypes.data_as(_u8p), *pix.shape)
    return out


def homotopic_thicken(img, allowed, priority, fg: int = 8, max_iter=None):
    """topo.py:317-354 (padded complement thinned under adj.dual())."""
    pix, pp = _u8(img)
    allowed, ap = _u8(allowed)
    prio, prp = _i64(priority)
    out = np.empty_like(pix)
    _load().orc_homotopic_thicken(pp, ap, prp, fg, -1 if max_iter is None else int(max_iter),
                                  out.ctypes.data_as(_u8p), *pix.shape)
    return out


def homotopic_cutting(img, keep, r, fg: int = 8):
    """smoothing.py:127-135"""
    pix, pp = _u8(img)
    keep, kp = _u8(keep)
    out = np.empty_like(pix)
    _load().orc_cutting(pp, kp, int(r), fg, out.ctypes.data_as(_u8p), *pix.shape)
    return out


def homotopic_filling(img, avoid, r, fg: int = 8):
    """smoothing.py:138-146"""
    pix, pp = _u8(img)
    avoid, ap = _u8(avoid)
    out = np.empty_like(pix)
    _load().orc_filling(pp, ap, int(r), fg, out.ctypes.data_as(_u8p), *pix.shape)
    return out


def hasf(img, r_max: int, fg: int = 8, keep=None, avoid=None):
    """smoothing.py:187-212"""
    pix, pp = _u8(img)
    kp = ap = None
    if keep is not None:
        keep = np.ascontiguousarray(keep, np.uint8)
        kp = keep.ctypes.data_as(_u8p)
    if avoid is not None:
        avoid = np.ascontiguousarray(avoid, np.uint8)
        ap = avoid.ctypes.data_as(_u8p)
    out = np.empty_like(pix)
    _load().orc_hasf(pp, kp, ap, int(r_max), fg, out.ctypes.data_as(_u8p), *pix.shape)
    return out


def hasf_batch(imgs, r_max: int, fg: int = 8, keep=None, avoid=None, threads: int | None = None):
    """smoothing.py:187-212 applied to every image of an [n,h,w] batch, images
    spread over `threads` host threads (independent units, no shared state)."""
    imgs = np.ascontiguousarray(imgs, np.uint8)
    n, h, w = imgs.shape
    out = np.empty_like(imgs)
    kp = ap = None
    if keep is not None:
        keep = np.ascontiguousarray(keep, np.uint8)
        kp = keep.ctypes.data_as(_u8p)
    if avoid is not None:
        avoid = np.ascontiguousarray(avoid, np.uint8)
        ap = avoid.ctypes.data_as(_u8p)
    _load().orc_hasf_batch(imgs.ctypes.data_as(_u8p), kp, ap, n, h, w, int(r_max), fg,
                           out.ctypes.data_as(_u8p), int(threads or os.cpu_count() or 1))
    return out


# ---- topology verifier (grid.py:93-128; scipy.ndimage.label as in grid.py:108) ----

def component_count(img, n: int = 8) -> int:
    from scipy import ndimage
    st = np.ones((3, 3), bool) if n == 8 else np.array([[0, 1, 0], [1, 1, 1], [0, 1, 0]], bool)
    return int(ndimage.label(np.asarray(img, np.uint8), structure=st)[1])


def background_component_count(img, n: int = 4) -> int:
    pix = np.asarray(img, np.uint8)
    padded = np.zeros((pix.shape[0] + 2, pix.shape[1] + 2), np.uint8)
    padded[1:-1, 1:-1] = pix
    return component_count(padded ^ 1, n)


def topology_preserved(before, after, fg: int = 8) -> bool:
    return (component_count(before, fg) == component_count(after, fg)
            and background_component_count(before, 12 - fg) == background_component_count(after, 12 - fg))


__all__ = [
    "build", "inf_value", "sep", "edt_squared", "edt_phase1_columns", "edt_phase2_rows",
    "border_distances_sq", "background_distances", "dilate", "erode", "luts",
    "neighborhood_codes", "simple_point_mask", "homotopic_thin", "homotopic_thicken",
    "homotopic_cutting", "homotopic_filling", "hasf", "hasf_batch", "component_count",
    "background_component_count", "topology_preserved",
]
