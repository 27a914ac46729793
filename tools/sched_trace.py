"""Schedule trace of fused launches (ts_set_trace) under several segment
settings, same process / same box: per setting the launch time, makespan,
busy time per SM, waits for predecessor segments, the idle tail when the
queue drains, mean task length per segment index, and the per-image work
(sum of its segments) against whole-image tasks.

    python tools/sched_trace.py --config c1 --settings 0:0,4:2,2:0 [--repeat 3]
"""
import argparse
import json
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

from paper_1603_09337_b200 import workloads as W  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="c1")
    ap.add_argument("--settings", default="0:0,4:2")
    ap.add_argument("--repeat", type=int, default=3)
    ap.add_argument("--n", type=int, default=0)
    a = ap.parse_args()
    import torch
    import paper_1603_09337_b200 as P
    from paper_1603_09337_b200 import _lib
    lib = _lib.load()
    cfg = W.CONFIGS[a.config]
    n = a.n or cfg.n
    x = torch.from_numpy(W.config_batch(cfg, 0, n)).cuda()
    adj = P.ADJ_84 if cfg.fg == 8 else P.ADJ_48
    cap = n * 64
    tr = torch.zeros((cap, 7), dtype=torch.int64, device="cuda")
    ref_out = P.hasf_batch(x, cfg.r_max, adj)
    out = {}
    for setting in a.settings.split(","):
        seg, fine = (int(v) for v in setting.split(":"))
        lib.ts_set_segment_stages(seg)
        lib.ts_set_segment_fine(fine)
        P.hasf_batch(x, cfg.r_max, adj)
        rows = []
        for rep in range(a.repeat):
            tr.zero_()
            lib.ts_set_trace(tr.data_ptr(), cap)
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            y = P.hasf_batch(x, cfg.r_max, adj)
            e1.record()
            torch.cuda.synchronize()
            lib.ts_set_trace(None, 0)
            assert torch.equal(y, ref_out)
            t = tr.cpu().numpy()
            t = t[t[:, 6] > 0]
            nseg = len(t) // n
            t0 = t[:, 1].min()
            sm, grab, ready, end = t[:, 0], (t[:, 1] - t0) / 1e3, (t[:, 2] - t0) / 1e3, (t[:, 6] - t0) / 1e3
            ph = np.diff(t[:, 2:7], axis=1) / 1e3   # load, stages, store, stats+barrier+publish
            span = end.max()
            ctas = len(np.unique(sm))
            last = {}
            for s_, e_ in zip(sm, end):
                last[s_] = max(last.get(s_, 0), e_)
            dur = end - ready
            rows.append({"event_ms": round(e0.elapsed_time(e1), 4), "span_us": round(float(span), 1),
                         "busy_us_per_sm": round(float(dur.sum() / ctas), 1),
                         "wait_us_per_sm": round(float((ready - grab).sum() / ctas), 1),
                         "tail_idle_us_per_sm": round(float(sum(span - v for v in last.values()) / ctas), 1),
                         "image_work_us": round(float(dur.sum() / n), 1), "tasks": int(len(t)),
                         "phase_us_per_image": [round(float(v), 2) for v in ph.sum(axis=0) / n],
                         "seg_mean_us": [round(float(np.mean(dur[k * n:(k + 1) * n])), 1) for k in range(nseg)]})
        out[setting] = min(rows, key=lambda r: r["event_ms"])
    print(json.dumps(out, indent=1))


if __name__ == "__main__":
    main()
