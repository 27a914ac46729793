"""CPU-side checks of the product package: the C-ABI library loads and exports
every symbol include/toposmooth_b200.h declares, host tables match the
reference, the bit-sliced simple-point formula matches the LUT, and the
Python mirror raises the reference's ValueErrors before touching a device.
No device compute happens here."""

import ctypes
import os
import re

import numpy as np
import pytest

import oracle as O
import paper_1603_09337_b200 as P
from paper_1603_09337_b200 import _lib
from conftest import REPO, load_golden


def header_symbols():
    text = open(os.path.join(REPO, "include", "toposmooth_b200.h")).read()
    return sorted(set(re.findall(r"\b(ts_[a-z0-9_]+)\s*\(", text)))


def test_library_exports_every_header_symbol():
    lib = _lib.load()
    syms = header_symbols()
    assert len(syms) >= 20
    for s in syms:
        assert hasattr(lib, s), s
    assert set(syms) == set(_lib.SIGNATURES), set(syms) ^ set(_lib.SIGNATURES)


def test_library_is_sm100a_cubin():
    import subprocess
    res = subprocess.run(["/usr/local/cuda/bin/cuobjdump", "--list-elf", _lib.LIB_PATH],
                         capture_output=True, text=True)
    assert res.returncode == 0, res.stderr
    assert "sm_100a" in res.stdout


def test_version_and_limits():
    lib = _lib.load()
    assert lib.ts_version() == 100
    assert lib.ts_max_radius() == 16   # the fused single-launch path; larger radii run per stage


def test_segment_fine_knob_semantics():
    """ts_set_segment_fine: a value fixes the scheduler's fine tail (and returns
    the previous one), a negative value returns to per-problem tuning and leaves
    the stored default alone.  Host state only."""
    lib = _lib.load()
    base = lib.ts_set_segment_fine(-1)
    assert base >= 0
    assert lib.ts_set_segment_fine(3) == base
    assert lib.ts_set_segment_fine(-1) == 3
    assert lib.ts_set_segment_fine(base) == 3
    assert lib.ts_set_segment_fine(-1) == base


def test_connectivity_tables_match_reference():
    z = load_golden("lut")
    assert np.array_equal(P.T8_TABLE, z["T8"]) and np.array_equal(P.T4_TABLE, z["T4"])
    assert np.array_equal(P.SIMPLE_84, z["SIMPLE_84"]) and np.array_equal(P.SIMPLE_48, z["SIMPLE_48"])


def yokoi(code, fg):
    """numpy restatement of the engine's bit-sliced circuit (csrc/ts_common.cuh)."""
    b = [(code >> k) & 1 for k in range(8)]
    nw, n, ne, w, e, sw, s, se = b
    if fg == 8:
        t = [(1 - e) & (ne | n), (1 - n) & (nw | w), (1 - w) & (sw | s), (1 - s) & (se | e)]
    else:
        t = [e & (1 - (ne & n)), n & (1 - (nw & w)), w & (1 - (sw & s)), s & (1 - (se & e))]
    return sum(t) == 1


def test_bitsliced_formula_equals_lut():
    _, _, s84, s48 = O.luts()
    for c in range(256):
        assert yokoi(c, 8) == bool(s84[c]), c
        assert yokoi(c, 4) == bool(s48[c]), c


def test_connectivity_numbers_host():
    img = np.zeros((3, 3), np.uint8)
    img[1, 1] = img[1, 2] = 1
    assert tuple(P.connectivity_numbers(img, (1, 1), P.ADJ_84)) == (1, 1, True)
    assert tuple(P.connectivity_numbers(np.ones((3, 3), np.uint8), (1, 1))) == (1, 0, False)
    with pytest.raises(ValueError):
        P.connectivity_numbers(np.zeros((3, 3), np.uint8), (1, 3))


def test_is_simple_all_256_window_oracle():
    # before/after window component counting (reference tests/oracles.py:81-99)
    from scipy import ndimage
    st = {4: np.array([[0, 1, 0], [1, 1, 1], [0, 1, 0]], bool), 8: np.ones((3, 3), bool)}
    offs = ((-1, -1), (-1, 0), (-1, 1), (0, -1), (0, 1), (1, -1), (1, 0), (1, 1))
    for mask in range(256):
        img = np.zeros((3, 3), np.uint8)
        img[1, 1] = 1
        for k, (dr, dc) in enumerate(offs):
            if (mask >> k) & 1:
                img[1 + dr, 1 + dc] = 1
        for adj in (P.ADJ_84, P.ADJ_48):
            after = img.copy()
            after[1, 1] = 0
            fg = ndimage.label(img, st[adj.fg])[1] == ndimage.label(after, st[adj.fg])[1]
            bg = ndimage.label(1 - img, st[adj.bg])[1] == ndimage.label(1 - after, st[adj.bg])[1]
            assert P.is_simple(img, (1, 1), adj) == (fg and bg), (mask, adj)


def test_validation_errors_match_reference():
    img = np.zeros((6, 6), np.uint8)
    img[2, 2] = 1
    with pytest.raises(ValueError, match="binary image pixels"):
        P.smooth(np.full((3, 3), 2, np.uint8), 1)
    with pytest.raises(ValueError, match="2D image"):
        P.smooth(np.zeros((2, 2, 2), np.uint8), 1)
    with pytest.raises(ValueError, match="2D image"):
        P.smooth(np.zeros((0, 3), np.uint8), 1)
    with pytest.raises(ValueError, match="radius"):
        P.hasf(img, P.SmoothingConfig(r_max=-1))
    with pytest.raises(ValueError, match="workers"):
        P.hasf(img, P.SmoothingConfig(r_max=1, workers=0))
    with pytest.raises(ValueError, match="scheduler"):
        P.hasf(img, P.SmoothingConfig(r_max=1, scheduler="fair"))
    keep = np.zeros_like(img)
    keep[2, 2] = 1
    with pytest.raises(ValueError, match="overlap"):
        P.hasf(img, P.SmoothingConfig(r_max=1, keep=keep, avoid=keep.copy()))
    bad_keep = np.zeros_like(img)
    bad_keep[0, 0] = 1
    with pytest.raises(ValueError, match="keep-constraint"):
        P.hasf(img, P.SmoothingConfig(r_max=1, keep=bad_keep))
    with pytest.raises(ValueError, match="avoid-constraint"):
        P.hasf(img, P.SmoothingConfig(r_max=1, avoid=keep))
    with pytest.raises(ValueError, match="match the input shape"):
        P.hasf(img, P.SmoothingConfig(r_max=1, keep=np.zeros((5, 5), np.uint8)))
    with pytest.raises(ValueError):
        P.homotopic_thin(img, bad_keep, np.zeros((6, 6), np.int64))
    with pytest.raises(ValueError):
        P.homotopic_thin(img, np.zeros((5, 6), np.uint8), np.zeros((6, 6), np.int64))
    with pytest.raises(ValueError):
        P.homotopic_thin(img, np.zeros_like(img), -np.ones((6, 6), np.int64))
    with pytest.raises(ValueError):
        P.homotopic_thicken(np.ones((3, 3), np.uint8), np.zeros((3, 3), np.uint8), np.zeros((3, 3), np.int64))
    centre = np.zeros((5, 5), np.uint8)
    centre[2, 2] = 1
    with pytest.raises(ValueError):
        P.homotopic_cutting(np.zeros((5, 5), np.uint8), centre, 1)
    with pytest.raises(ValueError):
        P.homotopic_filling(np.ones((4, 4), np.uint8), np.eye(4, dtype=np.uint8), 1)
    with pytest.raises(ValueError):
        P.edt_squared(img, workers=0)
    with pytest.raises(ValueError):
        P.edt_squared(img, scheduler="fifo")
    with pytest.raises(ValueError):
        P.dilate(img, -1)
    with pytest.raises(ValueError):
        P.Adjacency(6)


def test_host_scalar_helpers():
    z = load_golden("sep")
    for args, val in zip(z["args"], z["vals"]):
        assert P.sep(*map(int, args)) == int(val)
    with pytest.raises(ValueError):
        P.sep(3, 3, 0, 0)
    with pytest.raises(ValueError):
        P.sep(0, 1, -1, 0)
    assert P.inf_value((5, 4)) == 42
    assert P.ADJ_84.dual() == P.ADJ_48 and P.ADJ_48.bg == 8
    assert P.neighbors((0, 0), (3, 3), 4) == [(0, 1), (1, 0)]


def test_device_calls_fail_loudly_without_gpu():
    import torch
    if torch.cuda.is_available():
        pytest.skip("a GPU is present")
    with pytest.raises(RuntimeError, match="CUDA"):
        P.smooth(np.zeros((4, 4), np.uint8), 1)
    with pytest.raises(RuntimeError, match="CUDA"):
        P.edt_squared(np.zeros((4, 4), np.uint8))


def test_package_import_maps_no_native_library():
    """Importing the package (e.g. for its generators, as bench.py's reference
    arm does) must not map libtoposmooth_b200.so; the host-side tables equal
    the library's."""
    import subprocess
    import sys
    code = ("import paper_1603_09337_b200 as P\n"
            "print(any('libtoposmooth' in l for l in open('/proc/self/maps')))\n")
    res = subprocess.run([sys.executable, "-c", code], capture_output=True, text=True, cwd=REPO, timeout=300)
    assert res.stdout.strip().splitlines()[-1] == "False", res.stderr
    from paper_1603_09337_b200 import topo
    for a, b in zip(topo.native_tables(), (topo.T8_TABLE, topo.T4_TABLE, topo.SIMPLE_84, topo.SIMPLE_48)):
        assert np.array_equal(a, b)
