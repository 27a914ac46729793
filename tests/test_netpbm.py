"""netpbm I/O and the CLI's host logic against bytes / messages produced by
the reference (tests/golden/make_golden.py gen_netpbm); the device P4 path
and the CLI on the GPU are in test_gpu_parity.py."""

import numpy as np
import pytest

import paper_1603_09337_b200 as P
from paper_1603_09337_b200 import cli
from conftest import load_golden


def test_pbm_write_bytes_and_read_back(tmp_path):
    z = load_golden("netpbm")
    path = tmp_path / "x.pbm"
    for i in range(int(z["pbm_count"])):
        img = z[f"pbm{i}_img"]
        for fmt in ("P1", "P4"):
            P.write_pbm(img, path, format=fmt)
            assert path.read_bytes() == z[f"pbm{i}_{fmt}"].tobytes(), (i, fmt)
            assert np.array_equal(P.read_pbm(path), img)
            r = P.read_pbm_raster(path)
            assert (r.h, r.w, r.magic) == (img.shape[0], img.shape[1], fmt.encode())
            assert np.array_equal(r.unpack(), img)
            P.write_pbm_raster(r, tmp_path / "y.pbm", format=fmt)
            assert (tmp_path / "y.pbm").read_bytes() == z[f"pbm{i}_{fmt}"].tobytes()


def test_p4_padding_bits_ignored_and_zeroed(tmp_path):
    path = tmp_path / "p.pbm"
    path.write_bytes(b"P4\n3 2\n\xff\x1f")   # padding bits set on read
    r = P.read_pbm_raster(path)
    assert np.array_equal(r.unpack(), [[1, 1, 1], [0, 0, 0]])
    P.write_pbm_raster(r, tmp_path / "q.pbm")
    assert (tmp_path / "q.pbm").read_bytes() == b"P4\n3 2\n\xe0\x00"


def test_pgm_bytes_match_reference(tmp_path):
    z = load_golden("netpbm")
    path = tmp_path / "d.pgm"
    for name in ("dist", "empty"):
        m = z[f"pgm_{name}_in"]
        for mode in ("root", "squared"):
            for fmt in ("P2", "P5"):
                P.write_pgm(m, path, mode=mode, format=fmt)
                assert path.read_bytes() == z[f"pgm_{name}_{mode}_{fmt}"].tobytes(), (name, mode, fmt)
                assert np.array_equal(P.read_pgm(path), z[f"pgm_{name}_{mode}_{fmt}_read"])
    with pytest.raises(ValueError):
        P.write_pgm(np.zeros((2, 2), np.int64), path, mode="cube")
    with pytest.raises(ValueError):
        P.write_pbm(np.zeros((2, 2), np.uint8), path, format="P9")


def test_malformed_files_same_errors_as_reference(tmp_path):
    z = load_golden("netpbm")
    path = tmp_path / "bad"
    for i in range(int(z["bad_count"])):
        raw = z[f"bad{i}_raw"].tobytes()
        path.write_bytes(raw)
        reader = P.read_pgm if raw[:2] in (b"P2", b"P5") else P.read_pbm
        msg = str(z[f"bad{i}_msg"])
        if msg:
            with pytest.raises(P.NetpbmError) as e:
                reader(path)
            assert str(e.value) == msg, (raw, msg)
        else:
            assert np.array_equal(np.asarray(reader(path), np.int64).reshape(-1), z[f"bad{i}_out"])


def test_cli_argument_errors(tmp_path, capsys):
    assert cli.main([]) == 1
    assert cli.main(["--help"]) == 0
    assert cli.main(["frobnicate"]) == 1
    assert "unknown command" in capsys.readouterr().err
    assert cli.main(["smooth", str(tmp_path / "missing.pbm"), str(tmp_path / "o.pbm")]) == 1
    assert "error:" in capsys.readouterr().err
    img = tmp_path / "a.pbm"
    P.write_pbm(np.ones((4, 4), np.uint8), img)
    assert cli.main(["benchmark", str(img), "--workers-list", "0"]) == 1
    assert "positive integers" in capsys.readouterr().err
    assert cli.main(["benchmark", str(img), "--scheduler-list", "fifo"]) == 1
    assert "unknown scheduler" in capsys.readouterr().err
    assert cli.main(["benchmark", str(img), "--reps", "0"]) == 1
    assert cli.main(["smooth", str(img), str(tmp_path / "o.pbm"), "--adj", "6,6"]) == 1
    assert cli.main(["smooth", str(img), str(tmp_path / "o.pbm"), "--device", "cpu"]) == 1
    other = tmp_path / "b.pbm"
    P.write_pbm(np.zeros((5, 4), np.uint8), other)
    assert cli.main(["smooth", str(img), str(tmp_path / "o.pbm"), "--constraint-keep", str(other)]) == 1
    assert "keep-constraint is 4x5, image is 4x4" in capsys.readouterr().err
