"""Randomised parity stress (GPU): many random shapes / densities / radii
(incl. 17..20, the stage path) / adjacencies / constraints through
hasf_batch, the host entry and the P4 entry, under random kernel flavours,
team sizes (clusters, hierarchical, cooperative) and forced segmentation,
each checked bit-exact against the oracle.  Not part of the test suite.
    python tools/stress_parity.py [--cases 300] [--seed 0]"""
import argparse
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import oracle as O  # noqa: E402
import paper_1603_09337_b200 as P  # noqa: E402
from paper_1603_09337_b200 import _lib, workloads as W  # noqa: E402


def rand_img(rng, h, w):
    kind = rng.integers(0, 3)
    if kind == 0:
        return (rng.random((h, w)) < rng.uniform(0.05, 0.95)).astype(np.uint8)
    if kind == 1:   # blobs + noise
        return W.blob_image(h, w, int(rng.integers(1 << 30)), objects=int(rng.integers(1, 12)),
                            rad_lo=2, rad_hi=max(3, min(h, w) // 3), noise=float(rng.uniform(0, 0.1)))
    img = np.zeros((h, w), np.uint8)   # thin random walks
    y, x = rng.integers(0, h), rng.integers(0, w)
    for _ in range(int(rng.integers(10, 10 * (h + w)))):
        img[y, x] = 1
        y = int(np.clip(y + rng.integers(-1, 2), 0, h - 1))
        x = int(np.clip(x + rng.integers(-1, 2), 0, w - 1))
    return img ^ (rng.random((h, w)) < 0.02).astype(np.uint8)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--cases", type=int, default=300)
    ap.add_argument("--seed", type=int, default=0)
    ap.add_argument("--max-size", type=int, default=300, help="largest side (exclusive)")
    ap.add_argument("--max-r", type=int, default=8)
    a = ap.parse_args()
    rng = np.random.default_rng(a.seed)
    lib = _lib.load()
    bad = 0
    for i in range(a.cases):
        h, w = int(rng.integers(1, a.max_size)), int(rng.integers(1, a.max_size))
        n = int(rng.integers(1, 6 if a.max_size <= 300 else 3))
        fg = int(rng.choice([4, 8]))
        r = int(rng.integers(0, a.max_r + 1))
        imgs = np.stack([rand_img(rng, h, w) for _ in range(n)])
        keep = avoid = None
        if rng.random() < 0.3:
            keep = (imgs & (rng.random(imgs.shape) < 0.03)).astype(np.uint8)
            avoid = ((rng.random(imgs.shape) < 0.03) & (imgs == 0)).astype(np.uint8)
        if rng.random() < 0.03:   # radii above the fused kernel: the stage path
            r = int(rng.integers(17, 21))
        knobs = {"threads": int(rng.choice([0, 256, 512])), "team": int(rng.choice([0, 0, 0, 2, 3, 5, 8, 12])),
                 "fused": int(rng.choice([0, 1, 1])), "dense": int(rng.choice([2, 4, 8])),
                 "cluster": int(rng.choice([0, 1, 1, 2])), "seg_force": int(rng.random() < 0.3),
                 "seg": int(rng.choice([1, 2, 4, 8])), "fine": int(rng.choice([0, 1, 2, 3]))}
        lib.ts_set_cta_threads(knobs["threads"])
        lib.ts_set_team_size(knobs["team"])
        lib.ts_set_fused_prep(knobs["fused"])
        lib.ts_set_dense_divisor(knobs["dense"])
        lib.ts_set_cluster_teams(knobs["cluster"])
        lib.ts_set_segment_force(knobs["seg_force"])
        lib.ts_set_segment_stages(knobs["seg"])
        lib.ts_set_segment_fine(knobs["fine"])
        lib.ts_set_host_segments(knobs["seg"], knobs["fine"])
        adj = P.ADJ_84 if fg == 8 else P.ADJ_48
        want = O.hasf_batch(imgs, r, fg, keep=keep, avoid=avoid, threads=8)
        try:
            got = P.hasf_batch(imgs, r, adj, keep=keep, avoid=avoid)
        except RuntimeError as e:   # e.g. the 256-thread flavour does not fit
            if "does not fit" in str(e) or "needs the hot placement" in str(e):
                continue
            raise
        ok = np.array_equal(got, want)
        if knobs["team"] == 0:   # the host entry (packed / uint8 streaming / chunked), constraints too
            lib.ts_set_host_streaming(int(rng.choice([0, 1, 2])))
            hout = np.zeros_like(imgs)
            kp = None if keep is None else keep.ctypes.data
            ap_ = None if avoid is None else avoid.ctypes.data
            _lib.check(lib.ts_hasf_batch_host(imgs.ctypes.data, hout.ctypes.data, n, h, w, r, fg, kp, ap_, None))
            ok = ok and np.array_equal(hout, want)
        if rng.random() < 0.15:   # P4 rasters through the device bit rows
            pk = None if keep is None else np.packbits(keep, axis=2)
            pa = None if avoid is None else np.packbits(avoid, axis=2)
            got4 = P.hasf_p4(np.packbits(imgs, axis=2), w, r, adj, keep=pk, avoid=pa)
            ok = ok and np.array_equal(np.unpackbits(got4, axis=2)[:, :, :w], want)
        if not ok:
            bad += 1
            print("MISMATCH", i, dict(h=h, w=w, n=n, fg=fg, r=r, constraints=keep is not None, **knobs), flush=True)
    for f, v in (("ts_set_cta_threads", 0), ("ts_set_team_size", 0), ("ts_set_fused_prep", 1),
                 ("ts_set_dense_divisor", 4), ("ts_set_host_streaming", 1), ("ts_set_cluster_teams", 1),
                 ("ts_set_segment_force", 0), ("ts_set_segment_stages", 8), ("ts_set_segment_fine", 2)):
        getattr(lib, f)(v)
    lib.ts_set_host_segments(8, 0)
    print(f"stress: {a.cases} cases, {bad} mismatches")
    sys.exit(1 if bad else 0)


if __name__ == "__main__":
    main()
