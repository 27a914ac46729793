"""Barrier timeline of a cooperative-team launch (c3: one image over all SMs).
Needs a library built with -DTS_BAR_TRACE (TS_LIB_PATH=alt/bartrace.so): every
team barrier records %globaltimer at arrival and release per CTA.  Prints where
the launch's time goes: work between barriers, arrival skew (waiting for the
last CTA) and barrier latency (last arrival -> release), and which CTAs / SMs
arrive last.

    python -m paper_1603_09337_b200.build --define TS_BAR_TRACE --out alt/bartrace.so
    TS_LIB_PATH=alt/bartrace.so python tools/bar_trace.py --config c3
"""
import argparse
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1603_09337_b200 import workloads as W  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="c3")
    ap.add_argument("--cap", type=int, default=6000)
    a = ap.parse_args()
    import torch
    import paper_1603_09337_b200 as P
    from paper_1603_09337_b200 import _lib
    lib = _lib.load()
    cfg = W.CONFIGS[a.config]
    x = torch.from_numpy(W.config_batch(cfg, 0, 1)).cuda()
    adj = P.ADJ_84 if cfg.fg == 8 else P.ADJ_48
    G = torch.cuda.get_device_properties(0).multi_processor_count
    P.hasf_batch(x, cfg.r_max, adj)
    tr = torch.zeros((a.cap + 1, G, 2), dtype=torch.int64, device="cuda")
    lib.ts_set_trace(tr.data_ptr(), a.cap)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    P.hasf_batch(x, cfg.r_max, adj)
    e1.record()
    torch.cuda.synchronize()
    lib.ts_set_trace(None, 0)
    t = tr.cpu().numpy()
    smid = t[a.cap, :, 0]
    t = t[:a.cap]
    nb = int((t[:, 0, 0] > 0).sum())
    t = t[:nb].astype(np.float64)
    arr, rel = t[:, :, 0], t[:, :, 1]
    t0 = arr[0].min()
    arr, rel = (arr - t0) / 1e3, (rel - t0) / 1e3   # us
    print(f"launch {e0.elapsed_time(e1):.3f} ms, {nb} team barriers recorded, span {rel[-1].max() / 1e3:.3f} ms")
    last, first = arr.max(axis=1), arr.min(axis=1)
    lat = rel.min(axis=1) - last              # last arrival -> first release
    relspread = rel.max(axis=1) - rel.min(axis=1)
    work = arr[1:] - rel[:-1]                 # per CTA: release of barrier b-1 -> arrival at b
    wait = rel - arr                          # per CTA time inside the barrier
    print(f"per-CTA means over the launch (us): work {work.sum(axis=0).mean():.0f}  in-barrier {wait.sum(axis=0).mean():.0f}")
    print(f"  of the in-barrier time: latency (last arrival -> first release) {lat.sum():.0f}, "
          f"release spread (mean over CTAs) {(rel - rel.min(axis=1, keepdims=True)).sum(axis=0).mean():.0f}, "
          f"skew (mean CTA waiting for the last arrival) {(last[:, None] - arr).sum(axis=0).mean():.0f}")
    print(f"  per barrier: latency median {np.median(lat):.2f} us, p90 {np.percentile(lat, 90):.2f}; "
          f"arrival spread (last - first) median {np.median(last - first):.2f}, p90 {np.percentile(last - first, 90):.2f}, "
          f"sum {np.sum(last - first):.0f}")
    wmax, wmean = work.max(axis=1), work.mean(axis=1)
    print(f"  work per interval: mean-over-CTAs sum {wmean.sum():.0f} us, max-over-CTAs sum {wmax.sum():.0f} us "
          f"(imbalance {wmax.sum() / max(wmean.sum(), 1e-9):.2f}x)")
    # intervals by length of the slowest CTA
    edges = [0, 2, 5, 10, 20, 50, 100, 1e9]
    print("  intervals by slowest-CTA work (us): count, sum of max, sum of mean")
    for lo, hi in zip(edges[:-1], edges[1:]):
        m = (wmax >= lo) & (wmax < hi)
        print(f"    [{lo:>4g}, {hi:>4g}): {int(m.sum()):5d}  {wmax[m].sum():8.0f}  {wmean[m].sum():8.0f}")
    who = arr.argmax(axis=1)
    cnt = np.bincount(who, minlength=G)
    top = np.argsort(-cnt)[:8]
    print("  CTAs arriving last most often (rank:smid:count): " + "  ".join(f"{r}:{int(smid[r])}:{cnt[r]}" for r in top))
    # is lateness tied to the SM (position on the chip) or to the rank (its share of the image)?
    late = (arr - arr.mean(axis=1, keepdims=True)).mean(axis=0)
    order = np.argsort(-late)[:8]
    print("  mean lateness vs the barrier's mean arrival (us), worst ranks: " +
          "  ".join(f"{r}:{int(smid[r])}:{late[r]:.2f}" for r in order))
    print(f"  lateness by rank: std {late.std():.2f} us, min {late.min():.2f}, max {late.max():.2f}")
    # the barriers the team's first CTA arrives last at: by how much, and after how much work
    r0 = np.nonzero(who == 0)[0]
    r0 = r0[r0 > 0]
    if len(r0):
        second = np.sort(arr[r0], axis=1)[:, -2]
        gap = arr[r0, 0] - second
        w0 = work[r0 - 1, 0]
        wm = np.median(work[r0 - 1], axis=1)
        print(f"  rank 0 last at {len(r0)} barriers: ahead of it the next CTA by median {np.median(gap):.2f} us "
              f"(sum {gap.sum():.0f} us); its work before them median {np.median(w0):.2f} us vs the team's median "
              f"{np.median(wm):.2f} us")
        edges2 = [0, 2, 5, 10, 20, 50, 1e9]
        print("    by the team's median work in the interval (us): count, sum of rank 0's gap")
        for lo, hi in zip(edges2[:-1], edges2[1:]):
            m = (wm >= lo) & (wm < hi)
            print(f"      [{lo:>4g}, {hi:>4g}): {int(m.sum()):5d}  {gap[m].sum():8.0f}")
        d = np.diff(r0)
        print(f"    spacing of those barriers: median {np.median(d):.0f}, runs of consecutive ones {(d == 1).sum()}")


if __name__ == "__main__":
    main()
