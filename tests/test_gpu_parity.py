"""Parity of the CUDA path (through the C ABI) against the reference's golden
vectors and the CPU oracle.  Bit-exact everywhere (all arithmetic is integer)."""

import os

import numpy as np
import pytest

import oracle as O
import paper_1603_09337_b200 as P
from paper_1603_09337_b200 import _lib
from paper_1603_09337_b200 import workloads as W
from conftest import GOLDEN, golden_cases, random_image

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")
if not torch.cuda.is_available():  # pragma: no cover
    pytest.skip("needs a CUDA device", allow_module_level=True)


def test_circuit_equals_lut_on_device():
    import ctypes
    a, b = (ctypes.c_uint8 * 256)(), (ctypes.c_uint8 * 256)()
    _lib.check(_lib.load().ts_selftest_circuit(ctypes.addressof(a), ctypes.addressof(b)))
    assert np.array_equal(np.frombuffer(a, np.uint8), P.SIMPLE_84)
    assert np.array_equal(np.frombuffer(b, np.uint8), P.SIMPLE_48)


def test_edt_golden():
    for c in golden_cases("edt"):
        assert np.array_equal(P.edt_squared(c["img"]), c["out"]), c["name"]


def test_edt_phases():
    rng = np.random.default_rng(5)
    for _ in range(20):
        img = random_image(rng, int(rng.integers(1, 40)), int(rng.integers(1, 40)), rng.uniform(0.05, 0.9))
        g = P.edt_phase1_columns(img)
        assert np.array_equal(g, O.edt_phase1_columns(img))
        assert np.array_equal(P.edt_phase2_rows(g), O.edt_phase2_rows(g))
    img = np.zeros((3, 3), np.uint8)
    img[0, 0] = 1
    assert P.edt_phase2_rows(P.edt_phase1_columns(img))[2, 2] == 8


def test_edt_large_vs_oracle():
    for cfg in ("c1", "c4"):
        img = W.config_image(cfg, 3)
        assert np.array_equal(P.edt_squared(img), O.edt_squared(img))
        assert np.array_equal(P.background_distances(img), O.background_distances(img))


def test_morph_golden():
    for c in golden_cases("morph"):
        assert np.array_equal(P.background_distances(c["img"]), c["bgd"]), c["name"]
        assert np.array_equal(P.dilate(c["img"], c["r"]), c["dil"]), c["name"]
        assert np.array_equal(P.erode(c["img"], c["r"]), c["ero"]), c["name"]


def test_codes_and_simple_mask():
    rng = np.random.default_rng(11)
    for _ in range(20):
        img = random_image(rng, int(rng.integers(1, 50)), int(rng.integers(1, 50)), rng.uniform(0.1, 0.9))
        assert np.array_equal(P.neighborhood_codes(img), O.neighborhood_codes(img))
        for adj in (P.ADJ_84, P.ADJ_48):
            assert np.array_equal(P.simple_point_mask(img, adj), O.simple_point_mask(img, adj.fg))


def test_engine_golden():
    for c in golden_cases("engine"):
        adj = P.ADJ_84 if c["fg"] == 8 else P.ADJ_48
        mi = None if c["max_iter"] < 0 else c["max_iter"]
        assert np.array_equal(P.homotopic_thin(c["img"], c["keep"], c["pri"], adj, max_iter=mi), c["thin"]), c["name"]
        got = P.homotopic_thicken(c["img"], c["allowed"], c["pri"], adj, max_iter=mi)
        assert np.array_equal(got, c["thick"]), c["name"]


def test_engine_random_vs_oracle():
    rng = np.random.default_rng(12)
    for i in range(60):
        h, w = int(rng.integers(1, 80)), int(rng.integers(1, 80))
        fg = 8 if i % 2 else 4
        adj = P.ADJ_84 if fg == 8 else P.ADJ_48
        img = random_image(rng, h, w, rng.uniform(0.2, 0.9))
        keep = (img & random_image(rng, h, w, 0.05)).astype(np.uint8)
        pri = rng.integers(0, [3, 10, 1000][i % 3], (h, w)).astype(np.int64)
        mi = [None, 1, 3][i % 3]
        assert np.array_equal(P.homotopic_thin(img, keep, pri, adj, max_iter=mi),
                              O.homotopic_thin(img, keep, pri, fg, mi)), i
        allowed = (img | random_image(rng, h, w, 0.5)).astype(np.uint8)
        assert np.array_equal(P.homotopic_thicken(img, allowed, pri, adj, max_iter=mi),
                              O.homotopic_thicken(img, allowed, pri, fg, mi)), i


def test_halves_golden():
    for c in golden_cases("halves"):
        adj = P.ADJ_84 if c["fg"] == 8 else P.ADJ_48
        assert np.array_equal(P.homotopic_cutting(c["img"], c["keep"], c["r"], adj), c["cut"]), c["name"]
        assert np.array_equal(P.homotopic_filling(c["img"], c["avoid"], c["r"], adj), c["fill"]), c["name"]


def test_hasf_small_golden():
    for c in golden_cases("hasf_small"):
        adj = P.ADJ_84 if c["fg"] == 8 else P.ADJ_48
        keep = c["keep"] if c["keep"].any() else None
        avoid = c["avoid"] if c["avoid"].any() else None
        out = P.hasf(c["img"], P.SmoothingConfig(r_max=c["r"], adj=adj, keep=keep, avoid=avoid))
        assert np.array_equal(out, c["out"]), c["name"]


@pytest.mark.parametrize("name", ["c0_0", "c1_0", "c1_1", "c1_2", "c1_3", "c4_0", "c4_1", "c4_2", "c4_3", "c4_4",
                                  "c4_5", "c4_6", "c4_7", "jagged_disc_r5", "noisy_disc_r5", "c2_0"])
def test_hasf_config_golden(name):
    c = next(x for x in golden_cases("hasf_configs") if x["name"] == name)
    adj = P.ADJ_84 if c["fg"] == 8 else P.ADJ_48
    out = P.hasf(c["img"], P.SmoothingConfig(r_max=c["r"], adj=adj))
    assert np.array_equal(out, c["out"])


def test_hasf_batch_matches_single_and_golden():
    cases = [x for x in golden_cases("hasf_configs") if x["name"].startswith("c4_")]
    imgs = np.stack([c["img"] for c in cases])
    out = P.hasf_batch(torch.from_numpy(imgs).cuda(), 4, P.ADJ_48)
    assert out.is_cuda and out.dtype == torch.uint8
    for k, c in enumerate(cases):
        assert np.array_equal(out[k].cpu().numpy(), c["out"]), c["name"]
    host = P.hasf_batch_host(imgs, 4, P.ADJ_48)
    assert np.array_equal(host, out.cpu().numpy())


def test_hasf_batch_ragged_shapes_vs_oracle():
    rng = np.random.default_rng(13)
    for (h, w) in [(1, 1), (1, 77), (77, 1), (2, 2), (33, 31), (31, 33), (64, 96), (5, 200), (130, 65)]:
        imgs = np.stack([random_image(rng, h, w, rng.uniform(0.2, 0.8)) for _ in range(5)])
        for fg in (8, 4):
            adj = P.ADJ_84 if fg == 8 else P.ADJ_48
            got = P.hasf_batch(imgs, 3, adj)
            want = O.hasf_batch(imgs, 3, fg, threads=4)
            assert np.array_equal(got, want), (h, w, fg)


def test_hasf_batch_constraints_vs_oracle():
    rng = np.random.default_rng(14)
    imgs = np.stack([random_image(rng, 48, 70, 0.5) for _ in range(6)])
    keep = (imgs & (rng.random(imgs.shape) < 0.05)).astype(np.uint8)
    avoid = (((rng.random(imgs.shape) < 0.05)) & (imgs == 0)).astype(np.uint8)
    got = P.hasf_batch(imgs, 4, P.ADJ_84, keep=keep, avoid=avoid)
    want = O.hasf_batch(imgs, 4, 8, keep=keep, avoid=avoid, threads=4)
    assert np.array_equal(got, want)


def test_degenerate_images():
    for img in (np.zeros((64, 64), np.uint8), np.ones((64, 64), np.uint8), np.zeros((1, 1), np.uint8),
                np.ones((1, 1), np.uint8), np.ones((1, 40), np.uint8)):
        for r in (0, 1, 3):
            assert np.array_equal(P.smooth(img, r), O.hasf(img, r, 8))
    assert P.hasf_batch(np.zeros((0, 8, 8), np.uint8), 2).shape == (0, 8, 8)


def test_device_validation_errors():
    bad = np.zeros((2, 8, 8), np.uint8)
    bad[1, 3, 3] = 2
    with pytest.raises(ValueError, match="binary image pixels"):
        P.hasf_batch(torch.from_numpy(bad).cuda(), 1)
    imgs = np.zeros((2, 8, 8), np.uint8)
    keep = np.zeros_like(imgs)
    keep[0, 1, 1] = 1
    with pytest.raises(ValueError, match="keep-constraint"):
        P.hasf_batch(imgs, 1, keep=keep)
    imgs[1, 2, 2] = 1
    avoid = np.zeros_like(imgs)
    avoid[1, 2, 2] = 1
    with pytest.raises(ValueError, match="avoid-constraint"):
        P.hasf_batch(imgs, 1, avoid=avoid)
    # radii above the fused kernel (16) run the stage path: same validation
    with pytest.raises(ValueError, match="keep-constraint"):
        P.hasf_batch(np.zeros((2, 8, 8), np.uint8), 17, keep=keep)
    assert np.array_equal(P.smooth(np.zeros((8, 8), np.uint8), 17), np.zeros((8, 8), np.uint8))


def test_big_radii_golden():
    """Radii 17..25 (reference accepts any r >= 0, morph.py:18-22): the fused
    kernel up to 16, then per-stage launches (exact EDT -> stage mask -> the
    int64-priority engine), against reference goldens; also through the host,
    P4 and batched entries."""
    for c in golden_cases("hasf_big_r"):
        adj = P.ADJ_84 if c["fg"] == 8 else P.ADJ_48
        cfg = P.SmoothingConfig(r_max=c["r"], adj=adj, keep=c.get("keep"), avoid=c.get("avoid"))
        assert np.array_equal(P.hasf(c["img"], cfg), c["out"]), c["name"]
        r2 = 20 + int(c["name"][1:])
        z = np.zeros_like(c["img"])
        assert np.array_equal(P.homotopic_cutting(c["img"], z, r2, adj), c["cut"]), c["name"]
        assert np.array_equal(P.homotopic_filling(c["img"], z, r2, adj), c["fill"]), c["name"]
        if c.get("keep") is None and c.get("avoid") is None:
            imgs = np.stack([c["img"]] * 3)
            assert np.array_equal(P.hasf_batch_host(imgs, c["r"], adj)[2], c["out"]), c["name"]
            w = c["img"].shape[1]
            got = P.hasf_p4(np.packbits(imgs, axis=2), w, c["r"], adj)
            assert np.array_equal(np.unpackbits(got, axis=2)[1, :, :w], c["out"]), c["name"]
    img = W.config_image("c1", 7)[:200, :200].copy()
    assert np.array_equal(P.smooth(img, 18), O.hasf(img, 18, 8))


def test_topology_invariants_full_size_batches():
    """c1 / c4 shaped batches: component counts of X (fg-adjacency) and of the
    background with the window exterior attached (bg-adjacency) are preserved."""
    for cfg_name, count in (("c1", 8), ("c4", 32)):
        cfg = W.CONFIGS[cfg_name]
        imgs = W.config_batch(cfg, 100, count)
        out = P.hasf_batch(imgs, cfg.r_max, P.ADJ_84 if cfg.fg == 8 else P.ADJ_48)
        for a, b in zip(imgs, out):
            assert O.topology_preserved(a, b, cfg.fg)


def test_hasf_batch_vs_oracle_c1_c4_samples():
    for cfg_name, start, count in (("c1", 200, 3), ("c4", 500, 16)):
        cfg = W.CONFIGS[cfg_name]
        imgs = W.config_batch(cfg, start, count)
        got = P.hasf_batch(imgs, cfg.r_max, P.ADJ_84 if cfg.fg == 8 else P.ADJ_48)
        want = O.hasf_batch(imgs, cfg.r_max, cfg.fg)
        assert np.array_equal(got, want), cfg_name


def test_stats_are_reported():
    imgs = W.config_batch("c0", 0, 1)
    out, st = P.hasf_batch(imgs, 3, stats=True)
    assert st.shape == (1, 36) and st[0, 7] >= st[0, 4] + st[0, 5] > 0
    assert st[0, 2] == 12 and st[0, 0] > 0 and st[0, 1] >= st[0, 0] and st[0, 3] > 0


@pytest.fixture
def team_knob():
    lib = _lib.load()
    yield lib
    lib.ts_set_team_size(0)


@pytest.mark.parametrize("team,cluster", [(2, 1), (3, 1), (5, 1), (8, 1), (12, 2), (10, 2), (2, 0), (3, 0), (5, 0),
                                          (12, 0)])
def test_team_mode_vs_oracle(team_knob, team, cluster):
    """Teams of CTAs sharing one image through L2 (the large-image path),
    forced on small images so the oracle can check them: as thread-block
    clusters (hardware barrier, control block over DSMEM), as several
    clusters per team (teams > 8: hierarchical barrier) and as a cooperative
    launch with the global barrier."""
    team_knob.ts_set_team_size(team)
    old_cluster = team_knob.ts_set_cluster_teams(cluster)
    try:
        _team_cases(team)
    finally:
        team_knob.ts_set_cluster_teams(old_cluster)


def _team_cases(team):
    rng = np.random.default_rng(100 + team)
    for (h, w, fg, r) in [(160, 200, 8, 3), (97, 130, 4, 2), (64, 64, 8, 4)]:
        imgs = np.stack([random_image(rng, h, w, rng.uniform(0.3, 0.7)) for _ in range(3)])
        adj = P.ADJ_84 if fg == 8 else P.ADJ_48
        got = P.hasf_batch(imgs, r, adj)
        assert np.array_equal(got, O.hasf_batch(imgs, r, fg, threads=4)), (team, h, w, fg)
    img = random_image(rng, 70, 90, 0.6)
    keep = (img & random_image(rng, 70, 90, 0.05)).astype(np.uint8)
    pri = rng.integers(0, 7, (70, 90)).astype(np.int64)
    for mi in (None, 2):
        assert np.array_equal(P.homotopic_thin(img, keep, pri, P.ADJ_84, max_iter=mi),
                              O.homotopic_thin(img, keep, pri, 8, mi))
    allowed = (img | random_image(rng, 70, 90, 0.5)).astype(np.uint8)
    assert np.array_equal(P.homotopic_thicken(img, allowed, pri, P.ADJ_48),
                          O.homotopic_thicken(img, allowed, pri, 4, None))


def test_large_image_team_auto_vs_oracle():
    """One 2048^2 blob image (c3 generator statistics, cropped): hot planes do
    not fit one SM, a single image -> automatic team of CTAs."""
    img = W.blob_image(2048, 2048, 3000, objects=125, rad_lo=10, rad_hi=400, noise=0.05)
    out = P.hasf_batch(img[None], 4)
    assert np.array_equal(out[0], O.hasf(img, 4, 8))


def test_c3_full_size_topology():
    """Config c3 at full size (8192^2, r = 1..8): size-independent checks --
    topology invariants and the sandwich of the last filling (output differs
    from input only where smoothing acted)."""
    cfg = W.CONFIGS["c3"]
    img = W.config_image(cfg, 0)
    out, st = P.hasf_batch(img[None], cfg.r_max, stats=True)
    out = out[0]
    assert out.shape == img.shape and out.dtype == np.uint8 and out.max() <= 1
    assert O.topology_preserved(img, out, 8)
    assert st[0, 2] == 4 * cfg.r_max and st[0, 3] > 0


def test_host_entry_pinned_and_pageable_agree():
    imgs = W.config_batch("c4", 40, 12)
    want = O.hasf_batch(imgs, 4, 4, threads=4)
    pageable = P.hasf_batch_host(imgs, 4, P.ADJ_48)                 # staged copies
    pin_in = torch.from_numpy(imgs).pin_memory()
    pin_out = torch.empty_like(pin_in).pin_memory()
    _lib.check(_lib.load().ts_hasf_batch_host(pin_in.data_ptr(), pin_out.data_ptr(), 12, 256, 256, 4, 4, None, None,
                                              torch.cuda.current_stream().cuda_stream))   # zero-copy
    assert np.array_equal(pageable, want)
    assert np.array_equal(pin_out.numpy(), want)


@pytest.mark.parametrize("threads", [256, 512])
def test_kernel_flavours_vs_oracle(threads):
    """Both compiled flavours (512 threads x 1 CTA/SM, 256 x 2) on the same inputs."""
    lib = _lib.load()
    old = lib.ts_set_cta_threads(threads)
    try:
        rng = np.random.default_rng(300 + threads)
        for (h, w, fg, r) in [(256, 256, 4, 4), (200, 170, 8, 3), (33, 65, 8, 5)]:
            imgs = np.stack([random_image(rng, h, w, rng.uniform(0.3, 0.7)) for _ in range(4)])
            adj = P.ADJ_84 if fg == 8 else P.ADJ_48
            assert np.array_equal(P.hasf_batch(imgs, r, adj), O.hasf_batch(imgs, r, fg, threads=4)), (threads, h, w)
        imgs = W.config_batch("c4", 700, 8)
        assert np.array_equal(P.hasf_batch(imgs, 4, P.ADJ_48), O.hasf_batch(imgs, 4, 4, threads=4))
    finally:
        lib.ts_set_cta_threads(old)


def test_component_counts_vs_scipy():
    rng = np.random.default_rng(77)
    imgs = [random_image(rng, h, w, d) for (h, w, d) in [(1, 1, 1.0), (1, 1, 0.0), (5, 7, 0.5), (40, 33, 0.45),
                                                        (64, 64, 0.6), (97, 130, 0.3), (130, 65, 0.55)]]
    for img in imgs:
        for n in (4, 8):
            assert P.component_count(img, n) == O.component_count(img, n)
            assert P.component_count(img, n, foreground=False) == O.component_count(img ^ 1, n)
            assert P.background_component_count(img, n) == O.background_component_count(img, n)
    batch = W.config_batch("c4", 0, 16)
    fg, bg = P.topology_counts(batch, P.ADJ_48)
    for k in range(16):
        assert fg[k] == O.component_count(batch[k], 4) and bg[k] == O.background_component_count(batch[k], 8)


def test_topology_counts_full_size_outputs():
    img = W.config_image("c1", 9)
    out = P.smooth(img, 5)
    fi, bi = P.topology_counts(img[None])
    fo, bo = P.topology_counts(out[None])
    assert fi[0] == fo[0] == O.component_count(img, 8) and bi[0] == bo[0] == O.background_component_count(img, 4)


@pytest.mark.parametrize("fused", [1, 0])
def test_fused_and_two_phase_prep_vs_oracle(fused):
    """The fused prep + E-pass (rank slices in registers, neighbours by warp
    shuffle) and the two-phase prep / E-pass through rank planes give the
    oracle's output; shapes chosen on both sides of the fused path's
    eligibility (rows of 1, 2, 4, 8, 16 words; r up to 8; a 3-word row)."""
    lib = _lib.load()
    old = lib.ts_set_fused_prep(fused)
    try:
        rng = np.random.default_rng(500 + fused)
        for (h, w, fg, r) in [(96, 32, 8, 2), (64, 64, 4, 3), (80, 128, 8, 8), (40, 256, 8, 5), (50, 512, 4, 4),
                              (70, 90, 8, 6)]:
            imgs = np.stack([random_image(rng, h, w, rng.uniform(0.3, 0.7)) for _ in range(3)])
            adj = P.ADJ_84 if fg == 8 else P.ADJ_48
            assert np.array_equal(P.hasf_batch(imgs, r, adj), O.hasf_batch(imgs, r, fg, threads=4)), (fused, h, w, r)
        imgs = W.config_batch("c1", 1100, 2)
        assert np.array_equal(P.hasf_batch(imgs, 5), O.hasf_batch(imgs, 5, 8, threads=2))
        keep = (imgs & (rng.random(imgs.shape) < 0.02)).astype(np.uint8)
        avoid = ((rng.random(imgs.shape) < 0.02) & (imgs == 0)).astype(np.uint8)
        assert np.array_equal(P.hasf_batch(imgs, 3, P.ADJ_84, keep=keep, avoid=avoid),
                              O.hasf_batch(imgs, 3, 8, keep=keep, avoid=avoid, threads=2))
    finally:
        lib.ts_set_fused_prep(old)


@pytest.mark.parametrize("streaming", [1, 2, 0])
def test_streamed_host_entry_vs_device_path(streaming):
    """ts_hasf_batch_host: one launch gated on streamed input chunks (and
    chunk-gated copy-back) with host bit packing (1) or uint8 chunks (2), or
    the chunked pipeline (0) -- against the device-resident path, for batch
    sizes around the chunk size (16 images of 512^2), a single image, other
    shapes, ragged widths, keep / avoid constraints and invalid pixels (also
    in a chunk copied after the launch started)."""
    lib = _lib.load()
    old = lib.ts_set_host_streaming(streaming)
    try:
        stream = torch.cuda.current_stream().cuda_stream
        # (c2: team-sized images, one chunk per image, thread-block cluster teams gated on the chunks)
        for cfg, start, n in (("c1", 1200, 1), ("c1", 1210, 17), ("c1", 1230, 40), ("c2", 60, 3), ("c4", 4100, 70)):
            c = W.CONFIGS[cfg]
            imgs = W.config_batch(c, start, n)
            adj = P.ADJ_84 if c.fg == 8 else P.ADJ_48
            want = P.hasf_batch(imgs, c.r_max, adj)
            hin = torch.from_numpy(imgs).pin_memory()
            hout = torch.zeros_like(hin).pin_memory()
            _lib.check(lib.ts_hasf_batch_host(hin.data_ptr(), hout.data_ptr(), n, c.h, c.w, c.r_max, c.fg, None, None,
                                              stream))
            assert np.array_equal(hout.numpy(), want), (streaming, cfg, n)
        assert np.array_equal(want[:2], O.hasf_batch(imgs[:2], 4, 4, threads=2))
        rng = np.random.default_rng(77)
        imgs = np.stack([random_image(rng, 100, 96, 0.5) for _ in range(5)])
        keep = (imgs & (rng.random(imgs.shape) < 0.05)).astype(np.uint8)
        avoid = ((rng.random(imgs.shape) < 0.05) & (imgs == 0)).astype(np.uint8)
        out = np.zeros_like(imgs)
        _lib.check(lib.ts_hasf_batch_host(imgs.ctypes.data, out.ctypes.data, 5, 100, 96, 3, 8, keep.ctypes.data,
                                          avoid.ctypes.data, stream))
        assert np.array_equal(out, O.hasf_batch(imgs, 3, 8, keep=keep, avoid=avoid, threads=4))
        bad = imgs.copy()
        bad[2, 5, 5] = 7
        rc = lib.ts_hasf_batch_host(bad.ctypes.data, out.ctypes.data, 5, 100, 96, 3, 8, None, None, stream)
        assert rc == _lib.TS_ERR_VALUE and b"0 or 1" in lib.ts_last_error()
        for (h, w) in ((37, 45), (64, 33), (20, 300)):   # ragged widths (partial last word)
            imgs = np.stack([random_image(rng, h, w, 0.5) for _ in range(7)])
            out = np.zeros_like(imgs)
            _lib.check(lib.ts_hasf_batch_host(imgs.ctypes.data, out.ctypes.data, 7, h, w, 2, 4, None, None, stream))
            assert np.array_equal(out, O.hasf_batch(imgs, 2, 4, threads=4)), (streaming, h, w)
        # team-sized images (> 1024^2) with constraints, and an invalid pixel in the second of them
        imgs = np.stack([random_image(rng, 1100, 1040, 0.5) for _ in range(2)])
        keep = (imgs & (rng.random(imgs.shape) < 0.02)).astype(np.uint8)
        avoid = ((rng.random(imgs.shape) < 0.02) & (imgs == 0)).astype(np.uint8)
        out = np.zeros_like(imgs)
        _lib.check(lib.ts_hasf_batch_host(imgs.ctypes.data, out.ctypes.data, 2, 1100, 1040, 2, 8, keep.ctypes.data,
                                          avoid.ctypes.data, stream))
        assert np.array_equal(out, O.hasf_batch(imgs, 2, 8, keep=keep, avoid=avoid, threads=2)), streaming
        imgs[1, 1000, 1000] = 2
        rc = lib.ts_hasf_batch_host(imgs.ctypes.data, out.ctypes.data, 2, 1100, 1040, 2, 8, None, None, stream)
        assert rc == _lib.TS_ERR_VALUE and b"0 or 1" in lib.ts_last_error()
        big = W.config_batch("c1", 1300, 40)
        big[35, 100, 100] = 3   # lands in the third 16-image chunk
        hout = np.zeros_like(big)
        rc = lib.ts_hasf_batch_host(big.ctypes.data, hout.ctypes.data, 40, 512, 512, 5, 8, None, None, stream)
        assert rc == _lib.TS_ERR_VALUE and b"0 or 1" in lib.ts_last_error()
    finally:
        lib.ts_set_host_streaming(old)


# ---- large configs pinned to the reference (tests/golden/make_golden_large.py) ----
def _sha(a):
    import hashlib
    return hashlib.sha256(np.ascontiguousarray(a, np.uint8).tobytes()).hexdigest()


def _first_mismatch(got, bits):
    want = np.unpackbits(bits)[: got.size].reshape(got.shape)
    ys, xs = np.nonzero(got != want)
    return f"{len(ys)} pixels differ, first at ({ys[0]}, {xs[0]})" if len(ys) else "equal"


def test_c3_full_size_bit_exact():
    """Config c3 (8192^2, r = 1..8, (8,4)): the whole image bit-exact against
    the reference's own hasf output (SHA-256 + packed bits, generated by
    importing /root/reference, smoothing.py:187-212)."""
    z = np.load(os.path.join(GOLDEN, "large.npz"))
    cfg = W.CONFIGS["c3"]
    img = W.config_image(cfg, 0)
    assert _sha(img) == str(z["c3_0_in_sha"]), "generator drift: c3 input differs from the pinned one"
    out = P.hasf_batch(img[None], cfg.r_max)[0]
    assert _sha(out) == str(z["c3_0_out_sha"]), _first_mismatch(out, z["c3_0_out_bits"])


def test_c2_full_batch_bit_exact():
    """Config c2 as bench.py runs it: the full 32-image 2048^2 batch in one
    launch (team layout), four images pinned to the reference's hasf."""
    z = np.load(os.path.join(GOLDEN, "large.npz"))
    cfg = W.CONFIGS["c2"]
    imgs = W.config_batch(cfg, 0, cfg.n)
    out = P.hasf_batch(torch.from_numpy(imgs).cuda(), cfg.r_max).cpu().numpy()
    for i in (1, 7, 19, 31):
        assert _sha(imgs[i]) == str(z[f"c2_{i}_in_sha"]), f"generator drift on c2[{i}]"
        assert _sha(out[i]) == str(z[f"c2_{i}_out_sha"]), f"c2[{i}]: " + _first_mismatch(out[i], z[f"c2_{i}_out_bits"])


def test_segmented_scheduler_large_batch():
    """A c4 batch larger than one wave (600 images of 256^2, (4,8)) runs as
    (segment, image) tasks: identical to whole-image tasks, and to the oracle."""
    lib = _lib.load()
    imgs = torch.from_numpy(W.config_batch("c4", 4200, 600)).cuda()
    got = P.hasf_batch(imgs, 4, P.ADJ_48)
    old = lib.ts_set_segment_stages(0)
    try:
        whole = P.hasf_batch(imgs, 4, P.ADJ_48)
    finally:
        lib.ts_set_segment_stages(old)
    assert torch.equal(got, whole)
    sel = [0, 1, 299, 300, 599]
    host = imgs.cpu().numpy()[sel]
    assert np.array_equal(got.cpu().numpy()[sel], O.hasf_batch(host, 4, 4, threads=5))


@pytest.mark.parametrize("seg,fine", [(1, 0), (3, 1), (4, 2), (2, 5), (5, 0)])
def test_segmented_scheduler_forced_vs_oracle(seg, fine):
    """Forced segmentation on batches smaller than one wave: every task after
    the first of an image waits for its predecessor on another SM (the image
    and, mid-radius, the saved plane XS pass through global memory).  Both
    adjacencies, keep / avoid, radii 1..6, the streamed host entry."""
    lib = _lib.load()
    olds = (lib.ts_set_segment_stages(seg), lib.ts_set_segment_fine(fine), lib.ts_set_segment_force(1),
            lib.ts_set_host_segments(seg, fine))
    try:
        rng = np.random.default_rng(900 + seg * 10 + fine)
        for (h, w, fg, r) in [(96, 64, 8, 3), (128, 128, 4, 4), (70, 90, 8, 6), (33, 31, 4, 1)]:
            imgs = np.stack([random_image(rng, h, w, rng.uniform(0.3, 0.7)) for _ in range(6)])
            adj = P.ADJ_84 if fg == 8 else P.ADJ_48
            assert np.array_equal(P.hasf_batch(imgs, r, adj), O.hasf_batch(imgs, r, fg, threads=6)), (h, w, r)
            keep = (imgs & (rng.random(imgs.shape) < 0.03)).astype(np.uint8)
            avoid = ((rng.random(imgs.shape) < 0.03) & (imgs == 0)).astype(np.uint8)
            assert np.array_equal(P.hasf_batch(imgs, r, adj, keep=keep, avoid=avoid),
                                  O.hasf_batch(imgs, r, fg, keep=keep, avoid=avoid, threads=6)), (h, w, r)
        imgs = W.config_batch("c1", 1400, 20)
        want = O.hasf_batch(imgs, 5, 8, threads=8)
        assert np.array_equal(P.hasf_batch(imgs, 5), want)
        out = np.zeros_like(imgs)
        _lib.check(lib.ts_hasf_batch_host(imgs.ctypes.data, out.ctypes.data, 20, 512, 512, 5, 8, None, None,
                                          torch.cuda.current_stream().cuda_stream))
        assert np.array_equal(out, want)
        _, st = P.hasf_batch(imgs[:3], 5, stats=True)   # stats accumulate over the segments
        assert (st[:, 2] == 20).all()
    finally:
        lib.ts_set_segment_stages(olds[0])
        lib.ts_set_segment_fine(olds[1])
        lib.ts_set_segment_force(olds[2])
        lib.ts_set_host_segments(olds[3], 0)


def test_fine_tail_tuning_keeps_outputs():
    """The blocking entry tunes the segmented scheduler's fine tail over its
    first three launches of a problem (tail 2, 1, 2) and then keeps one: every
    one of those launches, and the non-blocking entry after them, returns the
    oracle's images."""
    lib = _lib.load()
    old_force = lib.ts_set_segment_force(1)
    lib.ts_set_segment_fine(-1)   # per-problem tuning on (earlier tests fixed the tail)
    try:
        rng = np.random.default_rng(77)
        imgs = np.stack([random_image(rng, 80, 100, rng.uniform(0.3, 0.7)) for _ in range(7)])
        want = O.hasf_batch(imgs, 4, 8, threads=7)
        x = torch.from_numpy(imgs).cuda()
        for _ in range(5):
            assert np.array_equal(P.hasf_batch(x, 4).cpu().numpy(), want)
        y, pending = P.hasf_batch(x, 4, blocking=False)
        pending.check()
        assert np.array_equal(y.cpu().numpy(), want)
    finally:
        lib.ts_set_segment_force(old_force)


# ---- netpbm P4 straight into the device layout, CLI on the device (row f2) ----
def test_p4_rows_round_trip_ragged_widths():
    lib = _lib.load()
    rng = np.random.default_rng(4040)
    st = torch.cuda.current_stream().cuda_stream
    for w in (1, 7, 8, 9, 31, 32, 33, 100, 513):
        h, n = 5, 3
        rb, ww = (w + 7) // 8, (w + 31) // 32
        img = (rng.random((n, h, w)) < 0.5).astype(np.uint8)
        p4 = np.packbits(img, axis=2)
        noisy = p4.copy()
        if w % 8:
            noisy[:, :, -1] |= np.uint8((1 << (8 - w % 8)) - 1)   # padding bits set: ignored
        d_p4 = torch.from_numpy(noisy).cuda()
        rows = torch.zeros((n, h, ww), dtype=torch.int32, device="cuda")
        _lib.check(lib.ts_p4_to_rows(d_p4.data_ptr(), rows.data_ptr(), n, h, w, st))
        r = rows.cpu().numpy().view(np.uint32)
        bits = ((r[..., None] >> np.arange(32, dtype=np.uint32)) & 1).reshape(n, h, ww * 32)[:, :, :w]
        assert np.array_equal(bits, img), w
        assert np.all((r[:, :, -1] >> np.uint32(w - 32 * (ww - 1))) == 0) or w % 32 == 0
        back = torch.full((n, h, rb), 0xAB, dtype=torch.uint8, device="cuda")
        _lib.check(lib.ts_rows_to_p4(rows.data_ptr(), back.data_ptr(), n, h, w, st))
        assert np.array_equal(back.cpu().numpy(), p4), w


def test_hasf_p4_matches_hasf():
    rng = np.random.default_rng(4041)
    imgs = W.config_batch("c1", 1500, 3)
    got = P.hasf_p4(np.packbits(imgs, axis=2), 512, 5)
    assert np.array_equal(np.unpackbits(got, axis=2)[:, :, :512], O.hasf_batch(imgs, 5, 8, threads=3))
    for (h, w, fg, r) in ((37, 45, 8, 3), (64, 33, 4, 2), (20, 300, 8, 4), (1, 1, 8, 1)):
        im = np.stack([random_image(rng, h, w, 0.5) for _ in range(4)])
        keep = (im & (rng.random(im.shape) < 0.05)).astype(np.uint8)
        avoid = ((rng.random(im.shape) < 0.05) & (im == 0)).astype(np.uint8)
        adj = P.ADJ_84 if fg == 8 else P.ADJ_48
        got = P.hasf_p4(np.packbits(im, axis=2), w, r, adj, keep=np.packbits(keep, axis=2),
                        avoid=np.packbits(avoid, axis=2))
        want = O.hasf_batch(im, r, fg, keep=keep, avoid=avoid, threads=4)
        assert np.array_equal(np.unpackbits(got, axis=2)[:, :, :w], want), (h, w)
        assert np.array_equal(got, np.packbits(want, axis=2))   # padding bits zero
    bad_keep = np.packbits(np.ones((1, 8, 8), np.uint8), axis=2)
    with pytest.raises(ValueError, match="keep-constraint pixels must be object pixels"):
        P.hasf_p4(np.packbits(np.zeros((1, 8, 8), np.uint8), axis=2), 8, 2, keep=bad_keep)
    big = W.config_batch("c4", 4300, 400)   # > one wave: segmented tasks on bit rows
    got = P.hasf_p4(np.packbits(big, axis=2), 256, 4, P.ADJ_48)
    assert np.array_equal(np.unpackbits(got, axis=2), P.hasf_batch(big, 4, P.ADJ_48))


def test_cli_smooth_and_benchmark_on_device(tmp_path, capsys):
    from paper_1603_09337_b200 import cli
    img = W.jagged_disc(256, 256, 90)
    src = tmp_path / "in.pbm"
    for fmt in ("P4", "P1"):
        P.write_pbm(img, src, format=fmt)
        out = tmp_path / f"out_{fmt}.pbm"
        assert cli.main(["smooth", str(src), str(out), "--radius", "4", "--verify", "--device", "cuda"]) == 0
        err = capsys.readouterr().err
        fb = [int(t) for t in err.split() if t.isdigit()]
        assert len(fb) == 4 and fb[0] == fb[1] and fb[2] == fb[3], err
        assert out.read_bytes()[:2] == fmt.encode()
        assert np.array_equal(P.read_pbm(out), O.hasf(img, 4, 8))
    P.write_pbm(img, src)
    assert cli.main(["smooth", str(src), str(tmp_path / "z.pbm"), "--radius", "0"]) == 0
    assert (tmp_path / "z.pbm").read_bytes() == src.read_bytes()
    keep = (img & (np.arange(img.size).reshape(img.shape) % 97 == 0)).astype(np.uint8)
    P.write_pbm(keep, tmp_path / "k.pbm")
    assert cli.main(["smooth", str(src), str(tmp_path / "c.pbm"), "--radius", "5", "--adj", "4,8",
                     "--constraint-keep", str(tmp_path / "k.pbm")]) == 0
    res = P.read_pbm(tmp_path / "c.pbm")
    assert np.array_equal(res, O.hasf(img, 5, 4, keep=keep)) and np.all(res[keep == 1] == 1)
    capsys.readouterr()
    assert cli.main(["benchmark", str(src), "--radius", "3", "--workers-list", "1,2", "--reps", "2"]) == 0
    lines = capsys.readouterr().out.strip().splitlines()
    assert lines[0] == "scheduler,workers,t_min_s,speedup,efficiency" and len(lines) == 3
    assert lines[1].startswith("nps,1,")


def test_constrained_hasf_at_scale_c1k():
    """Row f4: constrained HASF (keep / avoid control images, reference
    smoothing.py:197-206) on 16 full-size c1k images vs the oracle, in a
    batch larger than one wave (segmented) and through the streamed host
    entry with bit-packed constraint planes."""
    cfg = W.CONFIGS["c1k"]
    imgs = W.config_batch(cfg, 0, 300)
    keep, avoid = W.constraint_masks(cfg, imgs)
    got = P.hasf_batch(torch.from_numpy(imgs).cuda(), cfg.r_max, P.ADJ_84, keep=torch.from_numpy(keep).cuda(),
                       avoid=torch.from_numpy(avoid).cuda()).cpu().numpy()
    sel = list(range(8)) + list(range(292, 300))
    want = O.hasf_batch(imgs[sel], cfg.r_max, 8, keep=keep[sel], avoid=avoid[sel], threads=16)
    assert np.array_equal(got[sel], want)
    assert np.all(got[keep == 1] == 1) and np.all(got[avoid == 1] == 0)
    lib = _lib.load()
    n = 40
    out = np.zeros_like(imgs[:n])
    _lib.check(lib.ts_hasf_batch_host(imgs.ctypes.data, out.ctypes.data, n, cfg.h, cfg.w, cfg.r_max, 8,
                                      keep.ctypes.data, avoid.ctypes.data, torch.cuda.current_stream().cuda_stream))
    assert np.array_equal(out, got[:n])
    bad = keep[:n].copy()
    bad[33, 0, 0], bad[33, 0, 1] = 1, 2   # a non-binary constraint pixel in a late chunk
    rc = lib.ts_hasf_batch_host(imgs.ctypes.data, out.ctypes.data, n, cfg.h, cfg.w, cfg.r_max, 8, bad.ctypes.data,
                                avoid.ctypes.data, torch.cuda.current_stream().cuda_stream)
    assert rc == _lib.TS_ERR_VALUE and b"0 or 1" in lib.ts_last_error()
    k2 = keep[:n].copy()
    k2[5] |= (imgs[5] == 0)   # keep outside the object: the device-side check
    rc = lib.ts_hasf_batch_host(imgs.ctypes.data, out.ctypes.data, n, cfg.h, cfg.w, cfg.r_max, 8, k2.ctypes.data,
                                None, torch.cuda.current_stream().cuda_stream)
    assert rc == _lib.TS_ERR_VALUE and b"keep-constraint pixels must be object pixels" in lib.ts_last_error()


def test_nonblocking_batch_and_library_hygiene():
    """blocking=False: no synchronization inside, errors surface through the
    pending check; the device's default memory pool is left untouched (the
    library keeps a private pool)."""
    imgs = torch.from_numpy(W.config_batch("c4", 4500, 6)).cuda()
    out, pending = P.hasf_batch(imgs, 4, P.ADJ_48, blocking=False)
    pending.check()
    assert torch.equal(out, P.hasf_batch(imgs, 4, P.ADJ_48))
    bad = imgs.clone()
    bad[3, 7, 7] = 5
    out, pending = P.hasf_batch(bad, 4, P.ADJ_48, blocking=False)
    with pytest.raises(ValueError, match="0 or 1"):
        pending.check()
    import ctypes
    cudart = ctypes.CDLL("libcudart.so.12") if os.path.exists("/usr/local/cuda/lib64/libcudart.so.12") else None
    if cudart is not None:
        pool_h = ctypes.c_void_p()
        assert cudart.cudaDeviceGetDefaultMemPool(ctypes.byref(pool_h), 0) == 0
        thr = ctypes.c_uint64()
        assert cudart.cudaMemPoolGetAttribute(pool_h, 4, ctypes.byref(thr)) == 0   # ReleaseThreshold
        assert thr.value == 0


def _nccl_worker(port, q):
    import torch.distributed as dist
    from paper_1603_09337_b200.dist import hasf_sharded, max_over_ranks
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    torch.cuda.set_device(0)
    dist.init_process_group("nccl", rank=0, world_size=1)
    rng = np.random.default_rng(11)
    imgs = np.stack([random_image(rng, 40, 75, 0.5) for _ in range(5)])
    out = hasf_sharded(imgs, 3)                 # device path + bit-packed NCCL all-gather
    t = max_over_ranks(12.5)                    # device all-reduce (the bench's timing reduce)
    dist.barrier()
    dist.destroy_process_group()
    q.put((imgs, out, t))


def test_nccl_single_rank_sharded_gather():
    """The NCCL data path of dist.hasf_sharded / max_over_ranks on the device
    (one rank: this box has one GPU; world size 2 is covered with gloo on CPU)."""
    import socket
    import torch.multiprocessing as mp
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        port = s.getsockname()[1]
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    pr = ctx.Process(target=_nccl_worker, args=(port, q))
    pr.start()
    imgs, out, t = q.get(timeout=300)
    pr.join(timeout=60)
    assert pr.exitcode == 0
    assert np.array_equal(out, O.hasf_batch(imgs, 3, 8))
    assert t == 12.5


def test_registered_torch_op():
    """torch.ops.toposmooth_b200.hasf_batch: the CUDA implementation is the
    fused kernel, the fake implementation traces shape and dtype."""
    P.register_torch_ops()
    P.register_torch_ops()   # idempotent
    rng = np.random.default_rng(21)
    imgs = np.stack([random_image(rng, 50, 70, 0.5) for _ in range(3)])
    x = torch.from_numpy(imgs).cuda()
    y = torch.ops.toposmooth_b200.hasf_batch(x, 3)
    assert y.dtype == torch.uint8 and y.is_cuda
    assert np.array_equal(y.cpu().numpy(), O.hasf_batch(imgs, 3, 8))
    keep = (imgs & (rng.random(imgs.shape) < 0.05)).astype(np.uint8)
    y = torch.ops.toposmooth_b200.hasf_batch(x, 2, 4, torch.from_numpy(keep).cuda(), None)
    assert np.array_equal(y.cpu().numpy(), O.hasf_batch(imgs, 2, 4, keep=keep))
    with torch._subclasses.fake_tensor.FakeTensorMode():
        f = torch.ops.toposmooth_b200.hasf_batch(torch.empty((2, 8, 9), dtype=torch.uint8, device="cuda"), 1)
        assert tuple(f.shape) == (2, 8, 9) and f.dtype == torch.uint8
