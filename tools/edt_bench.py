"""Exact-EDT kernel timing (ts_edt_sq_batch) on config batches, and the
fraction of a fused HASF launch the same number of exact EDTs would cost
(why HASF uses the radius-clamped bit-parallel EDT).
    python tools/edt_bench.py [--config c1]"""
import argparse
import json
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1603_09337_b200 import _lib, workloads as W  # noqa: E402


def timed(fn, reps=5):
    fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        fn()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps


ap = argparse.ArgumentParser()
ap.add_argument("--config", default="c1")
ap.add_argument("--n", type=int, default=0)
a = ap.parse_args()
lib = _lib.load()
cfg = W.CONFIGS[a.config]
n = a.n or cfg.n
x = torch.from_numpy(W.config_batch(cfg, 0, n)).cuda()
out = torch.empty((n, cfg.h, cfg.w), dtype=torch.int64, device="cuda")
st = torch.cuda.current_stream().cuda_stream
t_edt = timed(lambda: _lib.check(lib.ts_edt_sq_batch(x.data_ptr(), out.data_ptr(), n, cfg.h, cfg.w, 1, st)))
res = {"config": cfg.name, "n": n, "edt_ms": t_edt,
       "edt_gpx_s": n * cfg.h * cfg.w / t_edt / 1e6,
       "edt_bytes_per_px_api": 1 + 8}
if hasattr(lib, "ts_hasf_batch"):
    o8 = torch.empty_like(x)
    t_h = timed(lambda: _lib.check(lib.ts_hasf_batch(x.data_ptr(), o8.data_ptr(), n, cfg.h, cfg.w, cfg.r_max, cfg.fg,
                                                       None, None, st, None)))
    res["hasf_ms"] = t_h
    res["exact_edts_per_hasf"] = 4 * cfg.r_max
    res["exact_edt_share_if_used"] = 4 * cfg.r_max * t_edt / t_h
print(json.dumps(res))
