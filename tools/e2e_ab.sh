#!/bin/bash
# GPU-box A/B of the streamed host entry: e2e ms per step (20 calls after 3 warm-ups) for each
# "stages:fine" host segmentation given (TS_SEG_STAGES_HOST / TS_SEG_FINE_HOST); CFG picks the config (c1)
for sf in "$@"; do
TS_SEG_STAGES_HOST=${sf%%:*} TS_SEG_FINE_HOST=${sf##*:} python - <<PY
import os, sys, torch, numpy as np
sys.path.insert(0, os.getcwd())
from paper_1603_09337_b200 import _lib, workloads as W
lib = _lib.load(); cfg = W.CONFIGS[os.environ.get("CFG", "c1")]
imgs = W.config_batch(cfg, 0, cfg.n); s = torch.cuda.current_stream()
x = torch.from_numpy(imgs).cuda(); out = torch.empty_like(x)
hin = torch.from_numpy(imgs).pin_memory(); hout = torch.empty_like(hin).pin_memory()
_lib.check(lib.ts_hasf_batch(x.data_ptr(), out.data_ptr(), cfg.n, cfg.h, cfg.w, cfg.r_max, cfg.fg, None, None, s.cuda_stream, None))
f = lambda: _lib.check(lib.ts_hasf_batch_host(hin.data_ptr(), hout.data_ptr(), cfg.n, cfg.h, cfg.w, cfg.r_max, cfg.fg, None, None, s.cuda_stream))
for _ in range(3): f()
torch.cuda.synchronize()
ts = []
for _ in range(20):
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(s); f(); e1.record(s); torch.cuda.synchronize(); ts.append(e0.elapsed_time(e1))
ok = np.array_equal(hout.numpy(), out.cpu().numpy())
print("host segments $sf: e2e mean %.3f ms  median %.3f  min %.3f  bit-exact vs device entry %s" % (np.mean(ts), np.median(ts), np.min(ts), ok))
PY
done
