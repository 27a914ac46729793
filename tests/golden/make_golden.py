"""Generate golden vectors from the REFERENCE implementation (run in the build
container only -- it imports /root/reference/pkg/src, which does not exist on
the GPU box).  The committed .npz files are what tests read.

    python tests/golden/make_golden.py            # writes tests/golden/*.npz

Families (each case stores its inputs and the reference output):
  lut      T8/T4/SIMPLE_84/SIMPLE_48 tables (topo.py:79-84)
  sep      sep() values incl. negative numerators (edt.py:31-42)
  edt      edt_squared on random sizes + degenerate images (edt.py:173-187)
  morph    background_distances / dilate / erode (morph.py:34-59)
  engine   homotopic_thin / homotopic_thicken with random priorities and
           max_iter (topo.py:303-342)
  halves   homotopic_cutting / homotopic_filling with constraints
           (smoothing.py:149-184)
  hasf     hasf on small random images (both adjacencies, keep/avoid) and on
           BASELINE config images c0, c1 (4 images), c2 (1 image), c4 (8
           images), plus the reference's own jagged_disc / noisy_disc inputs.
"""

from __future__ import annotations

import os
import sys
import time

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
REPO = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, "/root/reference/pkg/src")
sys.path.insert(0, REPO)

import toposmooth as ts  # noqa: E402
from toposmooth.topo import SIMPLE_48, SIMPLE_84, T4_TABLE, T8_TABLE  # noqa: E402

from paper_1603_09337_b200 import workloads as W  # noqa: E402


def pack(a):
    a = np.asarray(a, np.uint8)
    return np.packbits(a.reshape(-1)), np.array(a.shape, np.int64)


def rand_img(rng, h, w, density):
    return (rng.random((h, w)) < density).astype(np.uint8)


def adj_of(fg):
    return ts.ADJ_84 if fg == 8 else ts.ADJ_48


def gen_lut():
    np.savez_compressed(os.path.join(HERE, "lut.npz"), T8=T8_TABLE, T4=T4_TABLE,
                        SIMPLE_84=SIMPLE_84, SIMPLE_48=SIMPLE_48)


def gen_sep():
    rng = np.random.default_rng(7001)
    rows = [(0, 2, 0, 0), (0, 1, 0, 3), (1, 3, 2, 2), (1, 3, 0, 0), (0, 4, 7, 7), (0, 1, 4, 0)]
    for _ in range(300):
        i = int(rng.integers(0, 40))
        u = i + 1 + int(rng.integers(0, 40))
        rows.append((i, u, int(rng.integers(0, 30)), int(rng.integers(0, 30))))
    args = np.array(rows, np.int64)
    vals = np.array([ts.sep(*map(int, r)) for r in rows], np.int64)
    np.savez_compressed(os.path.join(HERE, "sep.npz"), args=args, vals=vals)


def gen_edt():
    rng = np.random.default_rng(7002)
    d = {}
    cases = []
    for _ in range(120):
        h, w = int(rng.integers(1, 48)), int(rng.integers(1, 48))
        cases.append(rand_img(rng, h, w, rng.uniform(0.01, 0.99)))
    for deg in (np.zeros((64, 64), np.uint8), np.ones((64, 64), np.uint8), np.zeros((1, 1), np.uint8),
                np.ones((1, 1), np.uint8), np.zeros((1, 37), np.uint8), rand_img(rng, 1, 97, 0.05),
                rand_img(rng, 97, 1, 0.05), rand_img(rng, 200, 3, 0.001)):
        cases.append(deg)
    for k, img in enumerate(cases):
        d[f"{k}_img"], d[f"{k}_shape"] = pack(img)
        d[f"{k}_out"] = ts.edt_squared(img)
    d["count"] = np.array(len(cases))
    np.savez_compressed(os.path.join(HERE, "edt.npz"), **d)


def gen_morph():
    rng = np.random.default_rng(7003)
    d = {}
    n = 60
    for k in range(n):
        h, w = int(rng.integers(1, 33)), int(rng.integers(1, 33))
        r = int(rng.integers(0, 6))
        img = rand_img(rng, h, w, rng.uniform(0.05, 0.95))
        d[f"{k}_img"], d[f"{k}_shape"] = pack(img)
        d[f"{k}_r"] = np.array(r)
        d[f"{k}_bgd"] = ts.background_distances(img)
        d[f"{k}_dil"] = pack(ts.dilate(img, r))[0]
        d[f"{k}_ero"] = pack(ts.erode(img, r))[0]
    d["count"] = np.array(n)
    np.savez_compressed(os.path.join(HERE, "morph.npz"), **d)


def gen_engine():
    rng = np.random.default_rng(7004)
    d = {}
    n = 160
    for k in range(n):
        h, w = int(rng.integers(1, 30)), int(rng.integers(1, 30))
        fg = 8 if k % 2 == 0 else 4
        img = rand_img(rng, h, w, rng.uniform(0.15, 0.9))
        keep = (img & rand_img(rng, h, w, 0.1)).astype(np.uint8)
        allowed = (img | rand_img(rng, h, w, 0.4)).astype(np.uint8)
        if k % 3 == 0:
            pri = ts.background_distances(img)
        elif k % 3 == 1:
            pri = rng.integers(0, 6, (h, w)).astype(np.int64)
        else:
            pri = rng.integers(0, 1 << 40, (h, w)).astype(np.int64)
        max_iter = [None, None, 0, 1, 2, 5][k % 6]
        d[f"{k}_img"], d[f"{k}_shape"] = pack(img)
        d[f"{k}_keep"] = pack(keep)[0]
        d[f"{k}_allowed"] = pack(allowed)[0]
        d[f"{k}_pri"] = pri
        d[f"{k}_fg"] = np.array(fg)
        d[f"{k}_max_iter"] = np.array(-1 if max_iter is None else max_iter)
        d[f"{k}_thin"] = pack(ts.homotopic_thin(img, keep, pri, adj_of(fg), max_iter=max_iter))[0]
        d[f"{k}_thick"] = pack(ts.homotopic_thicken(img, allowed, pri, adj_of(fg), max_iter=max_iter))[0]
    d["count"] = np.array(n)
    np.savez_compressed(os.path.join(HERE, "engine.npz"), **d)


def gen_halves():
    rng = np.random.default_rng(7005)
    d = {}
    n = 80
    for k in range(n):
        h, w = int(rng.integers(1, 40)), int(rng.integers(1, 40))
        fg = 8 if k % 2 == 0 else 4
        r = int(rng.integers(0, 5))
        img = rand_img(rng, h, w, rng.uniform(0.2, 0.8))
        keep = (img & rand_img(rng, h, w, 0.1)).astype(np.uint8)
        avoid = ((rand_img(rng, h, w, 0.1) == 1) & (img == 0)).astype(np.uint8)
        d[f"{k}_img"], d[f"{k}_shape"] = pack(img)
        d[f"{k}_keep"] = pack(keep)[0]
        d[f"{k}_avoid"] = pack(avoid)[0]
        d[f"{k}_r"] = np.array(r)
        d[f"{k}_fg"] = np.array(fg)
        d[f"{k}_cut"] = pack(ts.homotopic_cutting(img, keep, r, adj_of(fg)))[0]
        d[f"{k}_fill"] = pack(ts.homotopic_filling(img, avoid, r, adj_of(fg)))[0]
    d["count"] = np.array(n)
    np.savez_compressed(os.path.join(HERE, "halves.npz"), **d)


def gen_hasf_small():
    rng = np.random.default_rng(7006)
    d = {}
    n = 120
    for k in range(n):
        h, w = int(rng.integers(1, 45)), int(rng.integers(1, 70))
        fg = 8 if k % 2 == 0 else 4
        r_max = int(rng.integers(0, 7))
        img = rand_img(rng, h, w, rng.uniform(0.1, 0.9))
        if k % 4 == 3:
            keep = (img & rand_img(rng, h, w, 0.08)).astype(np.uint8)
            avoid = ((rand_img(rng, h, w, 0.08) == 1) & (img == 0)).astype(np.uint8)
        else:
            keep = np.zeros_like(img)
            avoid = np.zeros_like(img)
        out = ts.hasf(img, ts.SmoothingConfig(r_max=r_max, adj=adj_of(fg), keep=keep, avoid=avoid))
        d[f"{k}_img"], d[f"{k}_shape"] = pack(img)
        d[f"{k}_keep"] = pack(keep)[0]
        d[f"{k}_avoid"] = pack(avoid)[0]
        d[f"{k}_r"] = np.array(r_max)
        d[f"{k}_fg"] = np.array(fg)
        d[f"{k}_out"] = pack(out)[0]
    d["count"] = np.array(n)
    np.savez_compressed(os.path.join(HERE, "hasf_small.npz"), **d)


def gen_hasf_configs():
    """Full-size config images (reference hasf; the slow part)."""
    cases = []
    cases.append(("c0_0", W.config_image("c0", 0), 3, 8))
    for i in range(4):
        cases.append((f"c1_{i}", W.config_image("c1", i), 5, 8))
    for i in range(8):
        cases.append((f"c4_{i}", W.config_image("c4", i), 4, 4))
    cases.append(("jagged_disc_r5", W.jagged_disc(512, 512, 180), 5, 8))
    cases.append(("noisy_disc_r5", W.noisy_disc(512, 512, 180, np.random.default_rng(20240811), flip=0.02), 5, 8))
    if os.environ.get("GOLDEN_C2", "1") == "1":
        cases.append(("c2_0", W.config_image("c2", 0), 10, 8))
    d = {}
    names = []
    for name, img, r_max, fg in cases:
        t0 = time.perf_counter()
        out = ts.hasf(img, ts.SmoothingConfig(r_max=r_max, adj=adj_of(fg)))
        print(f"  {name}: {img.shape} r_max={r_max} fg={fg} ref {time.perf_counter() - t0:.1f}s", flush=True)
        d[f"{name}_img"], d[f"{name}_shape"] = pack(img)
        d[f"{name}_out"] = pack(out)[0]
        d[f"{name}_r"] = np.array(r_max)
        d[f"{name}_fg"] = np.array(fg)
        names.append(name)
    d["names"] = np.array(names)
    np.savez_compressed(os.path.join(HERE, "hasf_configs.npz"), **d)


def gen_netpbm():
    """netpbm.py: bytes the reference writes (P1 / P4 at ragged widths, PGM
    renderings), what it reads back, and its NetpbmError messages on
    malformed files."""
    import tempfile
    rng = np.random.default_rng(7009)
    d = {}
    tmp = tempfile.mkdtemp()
    path = os.path.join(tmp, "f")
    cases = [rand_img(rng, h, w, 0.5) for (h, w) in ((1, 1), (3, 7), (5, 8), (9, 13), (17, 40), (31, 70))]
    for i, img in enumerate(cases):
        d[f"pbm{i}_img"] = img
        for fmt in ("P1", "P4"):
            ts.write_pbm(img, path, format=fmt)
            d[f"pbm{i}_{fmt}"] = np.frombuffer(open(path, "rb").read(), np.uint8)
    d["pbm_count"] = np.array(len(cases))
    dist = ts.edt_squared(rand_img(rng, 12, 9, 0.2))
    dist_empty = ts.edt_squared(np.zeros((4, 5), np.uint8))
    for name, m in (("dist", dist), ("empty", dist_empty)):
        for mode in ("root", "squared"):
            for fmt in ("P2", "P5"):
                ts.write_pgm(m, path, mode=mode, format=fmt)
                d[f"pgm_{name}_{mode}_{fmt}"] = np.frombuffer(open(path, "rb").read(), np.uint8)
                d[f"pgm_{name}_{mode}_{fmt}_read"] = ts.read_pgm(path)
        d[f"pgm_{name}_in"] = m
    bad = [b"P3\n1 1\n0\n", b"P1\n2 2\n0 1 1\n", b"P4\n9 2\n\x00\x00\x00", b"P1\n0 2\n",
           b"P1\nx 2\n0 1", b"P1\n2 1\n0 2", b"P4\n8 1", b"P1 # c\n2 # c\n1\n01", b"P4\n3 1\n\xe0",
           b"P4\n3 2 \xff\x00", b"", b"P2\n2 1\n70000\n1 2\n", b"P5\n2 1\n255\n\x01"]
    msgs, imgs = [], []
    for raw in bad:
        open(path, "wb").write(raw)
        reader = ts.read_pgm if raw[:2] in (b"P2", b"P5") else ts.read_pbm
        try:
            out = reader(path)
            msgs.append("")
            imgs.append(np.asarray(out, np.int64).reshape(-1))
        except ts.NetpbmError as e:
            msgs.append(str(e))
            imgs.append(np.zeros(0, np.int64))
    d["bad_count"] = np.array(len(bad))
    for i, (raw, m, im) in enumerate(zip(bad, msgs, imgs)):
        d[f"bad{i}_raw"] = np.frombuffer(raw, np.uint8)
        d[f"bad{i}_msg"] = np.array(m)
        d[f"bad{i}_out"] = im
    np.savez_compressed(os.path.join(HERE, "netpbm.npz"), **d)


def gen_hasf_big_r():
    """Radii above the fused kernel's 16 (reference accepts any r >= 0,
    morph.py:18-22): hasf up to r_max 17..22 and single cutting / filling
    halves at r = 17..25, both adjacencies, with constraints."""
    rng = np.random.default_rng(7010)
    d, names = {}, []
    for i in range(6):
        h, w = int(rng.integers(40, 90)), int(rng.integers(40, 90))
        img = (rng.random((h, w)) < 0.55).astype(np.uint8)
        fg = 8 if i % 2 == 0 else 4
        r = 17 + i
        keep = (img & (rng.random((h, w)) < 0.02)).astype(np.uint8) if i % 3 == 0 else None
        avoid = (((rng.random((h, w)) < 0.02) & (img == 0)).astype(np.uint8)) if i % 3 == 1 else None
        out = ts.hasf(img, ts.SmoothingConfig(r_max=r, adj=adj_of(fg), keep=keep, avoid=avoid))
        k = f"h{i}"
        names.append(k)
        d[f"{k}_shape"] = np.array(img.shape)
        d[f"{k}_img"], _ = pack(img)
        d[f"{k}_out"], _ = pack(out)
        d[f"{k}_r"] = np.array(r)
        d[f"{k}_fg"] = np.array(fg)
        if keep is not None:
            d[f"{k}_keep"], _ = pack(keep)
        if avoid is not None:
            d[f"{k}_avoid"], _ = pack(avoid)
        cut = ts.homotopic_cutting(img, np.zeros_like(img), 20 + i, adj_of(fg))
        fil = ts.homotopic_filling(img, np.zeros_like(img), 20 + i, adj_of(fg))
        d[f"{k}_cut"], _ = pack(cut)
        d[f"{k}_fill"], _ = pack(fil)
    d["names"] = np.array(names)
    np.savez_compressed(os.path.join(HERE, "hasf_big_r.npz"), **d)


if __name__ == "__main__":
    which = sys.argv[1:] or ["lut", "sep", "edt", "morph", "engine", "halves", "hasf_small", "hasf_configs", "netpbm",
                             "hasf_big_r"]
    for name in which:
        t0 = time.perf_counter()
        globals()[f"gen_{name}"]()
        print(f"{name}: {time.perf_counter() - t0:.1f}s", flush=True)
