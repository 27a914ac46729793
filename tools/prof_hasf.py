"""Profiling driver: one fused-kernel launch over N images of a config, with
per-image engine stats and thread-0 phase cycle counters.  Used under ncu
(`-k regex:hasf_kernel -c 1`) and for quick phase breakdowns.

    python tools/prof_hasf.py --config c1 --n 148 [--smem-budget B] [--repeat 3]
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
    ap.add_argument("--n", type=int, default=148)
    ap.add_argument("--start", type=int, default=0)
    ap.add_argument("--smem-budget", type=int, default=-1)
    ap.add_argument("--repeat", type=int, default=1)
    ap.add_argument("--stats", type=int, default=1)
    ap.add_argument("--dense-div", type=int, default=0)
    ap.add_argument("--team", type=int, default=0)
    ap.add_argument("--threads", type=int, default=0)
    ap.add_argument("--cluster-teams", type=int, default=-1)
    ap.add_argument("--verify", type=int, default=0, help="images checked bit-exact vs the oracle")
    args = ap.parse_args()
    import torch
    import paper_1603_09337_b200 as P
    from paper_1603_09337_b200 import _lib
    cfg = W.CONFIGS[args.config]
    if args.smem_budget >= 0:
        _lib.load().ts_set_smem_budget(args.smem_budget)
    if args.dense_div > 0:
        _lib.load().ts_set_dense_divisor(args.dense_div)
    if args.team > 0:
        _lib.load().ts_set_team_size(args.team)
    if args.threads > 0:
        _lib.load().ts_set_cta_threads(args.threads)
    if args.cluster_teams >= 0:
        _lib.load().ts_set_cluster_teams(args.cluster_teams)
    args.n = args.n or cfg.n
    imgs_np = W.config_batch(cfg, args.start, args.n)
    imgs = torch.from_numpy(imgs_np).cuda()
    keep = avoid = None
    if cfg.constraints > 0:
        k_, a_ = W.constraint_masks(cfg, imgs_np, args.start)
        keep, avoid = torch.from_numpy(k_).cuda(), torch.from_numpy(a_).cuda()
    adj = P.ADJ_84 if cfg.fg == 8 else P.ADJ_48
    plan = np.zeros(6, np.int64)
    _lib.load().ts_hasf_plan(cfg.h, cfg.w, cfg.r_max, 0, 0, plan.ctypes.data)
    res = {"config": cfg.name, "n": args.n, "plan": plan.tolist(), "dense_div": args.dense_div, "team": args.team}
    for i in range(args.repeat):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        if args.stats:
            out, st = P.hasf_batch(imgs, cfg.r_max, adj, keep=keep, avoid=avoid, stats=True)
        else:
            out = P.hasf_batch(imgs, cfg.r_max, adj, keep=keep, avoid=avoid)
        e1.record()
        torch.cuda.synchronize()
        res[f"ms_{i}"] = e0.elapsed_time(e1)
    res["ms_min"] = min(res[f"ms_{i}"] for i in range(args.repeat))
    if args.verify:
        import oracle as O
        got = out.cpu().numpy()
        host = imgs.cpu().numpy()
        bad = [i for i in range(min(args.verify, args.n))
               if not np.array_equal(got[i], O.hasf(host[i], cfg.r_max, cfg.fg))]
        res["verify_bad"] = bad
    if args.stats:
        m = st.mean(axis=0)
        res.update({"sweeps": m[0], "passes": m[1], "calls": m[2], "flips": m[3],
                    "cyc_prep": m[4], "cyc_jacobi": m[5], "cyc_update": m[6], "cyc_total": m[7],
                    "cyc_total_max": int(st[:, 7].max()), "cyc_total_min": int(st[:, 7].min()),
                    "cyc_tiny": m[8], "n_tiny": m[9], "pass_tiny": m[10], "cyc_dense": m[11], "n_dense": m[12],
                    "pass_dense": m[13], "cyc_rank": m[14], "evals": m[15],
                                        "n_sp_small": m[16], "cyc_sp_small": m[17], "n_sp_big": m[18], "cyc_sp_big": m[19],
                    "x_tiny": m[28], "n_tinyreg": m[29], "y_pro": m[32], "y_top": m[33], "y_epi": m[34], "y_iter": m[35], "x_engine": m[30], "x_stage": m[31], "b_build": m[24], "b_sweep": m[25], "b_rebuild": m[26], "n_build": m[27],
                    "cyc_dpass1": m[20], "cyc_dcollect": m[21], "cyc_dlist": m[22], "d_listed": m[23]})
    print(json.dumps(res, default=float))


if __name__ == "__main__":
    main()
