"""Pins the CPU oracle (oracle/, test infrastructure) against golden vectors
produced by the imported reference (tests/golden/make_golden.py).  CPU only."""

import numpy as np
import pytest

import oracle as O
from conftest import golden_cases, load_golden


def test_lut_tables_match_reference():
    z = load_golden("lut")
    t8, t4, s84, s48 = O.luts()
    assert np.array_equal(t8, z["T8"]) and np.array_equal(t4, z["T4"])
    assert np.array_equal(s84, z["SIMPLE_84"]) and np.array_equal(s48, z["SIMPLE_48"])
    assert int(s84.sum()) == 116 and int(s48.sum()) == 116
    assert np.array_equal(s48, s84[np.arange(256) ^ 0xFF])


def test_lut_hex_known_answers():
    _, _, s84, s48 = O.luts()
    as_int = lambda a: sum(int(b) << i for i, b in enumerate(a))   # noqa: E731
    assert f"{as_int(s84):064x}" == "33ddcf0133ddcf01cc000000ccdd000133ddcf0133ddcf01cc00cf01ccddcfde"
    assert f"{as_int(s48):064x}" == "7bf3bb3380f3003380f3bbcc80f3bbcc8000bb330000003380f3bbcc80f3bbcc"


def test_sep_values():
    z = load_golden("sep")
    for args, val in zip(z["args"], z["vals"]):
        assert O.sep(*map(int, args)) == int(val)
    assert O.sep(0, 1, 4, 0) == -8   # negative numerator: floor, not truncation


def test_edt_golden():
    for c in golden_cases("edt"):
        assert np.array_equal(O.edt_squared(c["img"]), c["out"]), c["name"]


def test_edt_phases_known_answers():
    img = np.zeros((3, 1), np.uint8)
    img[0, 0] = 1
    assert O.edt_phase1_columns(img)[:, 0].tolist() == [0, 1, 2]
    img = np.zeros((5, 1), np.uint8)
    img[0, 0] = img[4, 0] = 1
    assert O.edt_phase1_columns(img)[:, 0].tolist() == [0, 1, 2, 1, 0]
    img = np.zeros((3, 3), np.uint8)
    img[0, 0] = 1
    assert O.edt_phase2_rows(O.edt_phase1_columns(img))[2, 2] == 8


def test_morph_golden():
    for c in golden_cases("morph"):
        assert np.array_equal(O.background_distances(c["img"]), c["bgd"]), c["name"]
        assert np.array_equal(O.dilate(c["img"], c["r"]), c["dil"]), c["name"]
        assert np.array_equal(O.erode(c["img"], c["r"]), c["ero"]), c["name"]


def test_engine_golden():
    for c in golden_cases("engine"):
        mi = None if c["max_iter"] < 0 else c["max_iter"]
        assert np.array_equal(O.homotopic_thin(c["img"], c["keep"], c["pri"], c["fg"], mi), c["thin"]), c["name"]
        assert np.array_equal(O.homotopic_thicken(c["img"], c["allowed"], c["pri"], c["fg"], mi), c["thick"]), c["name"]


def test_halves_golden():
    for c in golden_cases("halves"):
        assert np.array_equal(O.homotopic_cutting(c["img"], c["keep"], c["r"], c["fg"]), c["cut"]), c["name"]
        assert np.array_equal(O.homotopic_filling(c["img"], c["avoid"], c["r"], c["fg"]), c["fill"]), c["name"]


def test_hasf_small_golden():
    for c in golden_cases("hasf_small"):
        out = O.hasf(c["img"], c["r"], c["fg"], c["keep"], c["avoid"])
        assert np.array_equal(out, c["out"]), c["name"]


@pytest.mark.parametrize("name", ["c0_0", "c1_0", "c4_0", "c4_1", "jagged_disc_r5", "noisy_disc_r5"])
def test_hasf_config_golden(name):
    c = next(x for x in golden_cases("hasf_configs") if x["name"] == name)
    assert np.array_equal(O.hasf(c["img"], c["r"], c["fg"]), c["out"])


def test_hasf_batch_threads_match_serial():
    z = [c for c in golden_cases("hasf_configs") if c["name"].startswith("c4_")]
    imgs = np.stack([c["img"] for c in z])
    out = O.hasf_batch(imgs, 4, 4, threads=4)
    for k, c in enumerate(z):
        assert np.array_equal(out[k], c["out"]), c["name"]


def test_large_goldens_inputs_and_oracle_c2():
    """tests/golden/large.npz (reference hasf on c2 / c3 config images): the
    generators still reproduce the pinned inputs, and the oracle matches the
    reference on one full-size c2 image (2048^2, r = 1..10)."""
    import hashlib
    import os
    from conftest import GOLDEN
    from paper_1603_09337_b200 import workloads as W
    sha = lambda a: hashlib.sha256(np.ascontiguousarray(a, np.uint8).tobytes()).hexdigest()  # noqa: E731
    z = np.load(os.path.join(GOLDEN, "large.npz"))
    cfg = W.CONFIGS["c2"]
    for i in (1, 7, 19, 31):
        assert sha(W.config_image(cfg, i)) == str(z[f"c2_{i}_in_sha"])
    img = W.config_image(cfg, 31)
    assert sha(O.hasf(img, cfg.r_max, 8)) == str(z["c2_31_out_sha"])


def test_oracle_big_radii_golden():
    """Radii above 16 (reference hasf / homotopic_cutting / homotopic_filling)."""
    for c in golden_cases("hasf_big_r"):
        keep = c.get("keep")
        avoid = c.get("avoid")
        assert np.array_equal(O.hasf(c["img"], c["r"], c["fg"], keep=keep, avoid=avoid), c["out"]), c["name"]
