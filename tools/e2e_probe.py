"""Probe the host-buffer entry: H2D/D2H bandwidth of pinned buffers, and the
e2e time of ts_hasf_batch_host vs the device-resident kernel for a few sizes.
    python tools/e2e_probe.py"""
import os
import sys
import time

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1603_09337_b200 import _lib, workloads as W  # noqa: E402


def timed(fn, reps=5):
    s = torch.cuda.current_stream()
    fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(s)
    for _ in range(reps):
        fn()
    e1.record(s)
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps


lib = _lib.load()
cfg = W.CONFIGS["c1"]
for nbytes in (4 << 20, 64 << 20):
    h = torch.empty(nbytes, dtype=torch.uint8).pin_memory()
    d = torch.empty(nbytes, dtype=torch.uint8, device="cuda")
    t1 = timed(lambda: d.copy_(h, non_blocking=True))
    t2 = timed(lambda: h.copy_(d, non_blocking=True))
    print(f"{nbytes >> 20} MiB: H2D {nbytes / t1 / 1e6:.1f} GB/s  D2H {nbytes / t2 / 1e6:.1f} GB/s")
imgs = W.config_batch(cfg, 0, 256)
s = torch.cuda.current_stream()
for n in (16, 148, 256):
    x = torch.from_numpy(imgs[:n]).cuda()
    out = torch.empty_like(x)
    hin = torch.from_numpy(imgs[:n]).pin_memory()
    hout = torch.empty_like(hin).pin_memory()
    tk = timed(lambda: _lib.check(lib.ts_hasf_batch(x.data_ptr(), out.data_ptr(), n, 512, 512, 5, 8, None, None,
                                                     s.cuda_stream, None)))
    res = [f"n={n}: kernel {tk:.3f} ms"]
    for hs in (1, 0):
        lib.ts_set_host_streaming(hs)
        te = timed(lambda: _lib.check(lib.ts_hasf_batch_host(hin.data_ptr(), hout.data_ptr(), n, 512, 512, 5, 8,
                                                              None, None, s.cuda_stream)))
        assert np.array_equal(hout.numpy(), out.cpu().numpy())
        res.append(f"e2e(streaming={hs}) {te:.3f} ms")
    print("  ".join(res))

# segment settings (the streamed entry's fused launch is segmented too)
n = 256
x = torch.from_numpy(imgs).cuda()
out = torch.empty_like(x)
hin = torch.from_numpy(imgs).pin_memory()
hout = torch.empty_like(hin).pin_memory()
lib.ts_set_host_streaming(1)
for seg, fine in ((0, 0), (4, 0), (4, 2), (8, 0), (8, 2), (12, 0), (12, 4)):
    lib.ts_set_segment_stages(seg)
    lib.ts_set_segment_fine(fine)
    lib.ts_set_host_segments(seg, fine)
    tk = timed(lambda: _lib.check(lib.ts_hasf_batch(x.data_ptr(), out.data_ptr(), n, 512, 512, 5, 8, None, None,
                                                     s.cuda_stream, None)))
    te = timed(lambda: _lib.check(lib.ts_hasf_batch_host(hin.data_ptr(), hout.data_ptr(), n, 512, 512, 5, 8,
                                                          None, None, s.cuda_stream)))
    print(f"seg {seg}:{fine}: kernel {tk:.3f} ms  e2e {te:.3f} ms")
