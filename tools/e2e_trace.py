"""Host timeline of ts_hasf_batch_host for c1 (TS_HOST_TRACE=1): per chunk, when it was sent, when its
copy-back finished and when it was unpacked; with the device-resident kernel time beside it.
    TS_HOST_TRACE=1 python tools/e2e_trace.py"""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1603_09337_b200 import _lib, workloads as W  # noqa: E402

lib = _lib.load()
cfg = W.CONFIGS["c1"]
imgs = W.config_batch(cfg, 0, cfg.n)
s = torch.cuda.current_stream()
x = torch.from_numpy(imgs).cuda()
out = torch.empty_like(x)
hin = torch.from_numpy(imgs).pin_memory()
hout = torch.empty_like(hin).pin_memory()
for _ in range(3):
    _lib.check(lib.ts_hasf_batch(x.data_ptr(), out.data_ptr(), cfg.n, cfg.h, cfg.w, cfg.r_max, cfg.fg, None, None, s.cuda_stream, None))
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record(s)
_lib.check(lib.ts_hasf_batch(x.data_ptr(), out.data_ptr(), cfg.n, cfg.h, cfg.w, cfg.r_max, cfg.fg, None, None, s.cuda_stream, None))
e1.record(s)
torch.cuda.synchronize()
print("device-resident kernel: %.3f ms" % e0.elapsed_time(e1), file=sys.stderr)
for _ in range(4):
    _lib.check(lib.ts_hasf_batch_host(hin.data_ptr(), hout.data_ptr(), cfg.n, cfg.h, cfg.w, cfg.r_max, cfg.fg, None, None, s.cuda_stream))
