import os, sys, torch
sys.path.insert(0, os.getcwd())
from paper_1603_09337_b200 import _lib, workloads as W
lib = _lib.load()
cfg = W.CONFIGS["c1k"]
imgs = W.config_batch(cfg, 0, cfg.n)
k, a = W.constraint_masks(cfg, imgs, 0)
s = torch.cuda.current_stream()
hin = torch.from_numpy(imgs).pin_memory(); hk = torch.from_numpy(k).pin_memory(); ha = torch.from_numpy(a).pin_memory()
hout = torch.empty_like(hin).pin_memory()
for _ in range(4):
    _lib.check(lib.ts_hasf_batch_host(hin.data_ptr(), hout.data_ptr(), cfg.n, cfg.h, cfg.w, cfg.r_max, cfg.fg, hk.data_ptr(), ha.data_ptr(), s.cuda_stream))
