import os, sys, time, numpy as np, torch
sys.path.insert(0, os.getcwd())
import paper_1603_09337_b200 as P
from paper_1603_09337_b200 import _lib, workloads as W
lib=_lib.load()
s=torch.cuda.current_stream()
for cfgname, n in (("c2", 3), ("c2", 32), ("c3", 1)):
    cfg=W.CONFIGS[cfgname]
    imgs=W.config_batch(cfg, 0, n)
    x=torch.from_numpy(imgs).cuda()
    want=P.hasf_batch(x, cfg.r_max).cpu().numpy()
    hin=torch.from_numpy(imgs).pin_memory(); hout=torch.zeros_like(hin).pin_memory()
    f=lambda: _lib.check(lib.ts_hasf_batch_host(hin.data_ptr(), hout.data_ptr(), n, cfg.h, cfg.w, cfg.r_max, cfg.fg, None, None, s.cuda_stream))
    f(); torch.cuda.synchronize()
    ok=np.array_equal(hout.numpy(), want)
    ts=[]
    for _ in range(4):
        t=time.perf_counter(); f(); torch.cuda.synchronize(); ts.append((time.perf_counter()-t)*1e3)
    print(cfgname, n, "TS_STREAM_BIG", os.environ.get("TS_STREAM_BIG","1"), "ok", ok, "e2e ms min %.2f median %.2f" % (min(ts), np.median(ts)), "img/s %.1f" % (n/min(ts)*1e3), flush=True)
