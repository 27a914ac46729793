#!/usr/bin/env python
"""HASF throughput bench (BASELINE.json metric: images/s on a 512^2 batch,
% of the HBM roofline, vs the CPU reference).

  python bench.py [--gpus N --steps K --warmup W] [--config c1] [--impl ours|reference]

Default workload = config c1 (256 x 512x512 synthetic blob images, r = 1..5,
(8,4)).  A step = one hasf_batch over the rank's whole batch, inputs already
resident in HBM (value); e2e = the same through the C ABI's host-buffer entry
(ts_hasf_batch_host: pinned host -> device copy, kernel, device -> host copy
inside the timed region).  Multi-GPU (torchrun): every rank smooths its own
256 distinct images (weak scaling, no data-path collective); time = max over
ranks.  --impl reference times the CPU restatement of the reference (oracle/,
all host threads) on a bounded sample of the same workload.
"""

from __future__ import annotations

import argparse
import json
import os
import subprocess
import sys
import threading
import time

import numpy as np

REPO = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, REPO)



def _load_workloads():
    """The seeded generators, loaded by file path: the reference arm must not
    import the product package (nothing of ours may be mapped in its process)."""
    import importlib.util
    name = "_ts_bench_workloads"
    spec = importlib.util.spec_from_file_location(name, os.path.join(REPO, "paper_1603_09337_b200", "workloads.py"))
    mod = importlib.util.module_from_spec(spec)
    sys.modules[name] = mod
    spec.loader.exec_module(mod)
    return mod


W = _load_workloads()
REF_DIR = os.path.join(REPO, "baseline", "_ref")

METRIC = "HASF images/s (512^2 batch, 1 B200), % HBM roofline, vs CPU ref"
E2E_PATH = {True: "ts_hasf_batch_host (C ABI, pinned host buffers; one fused launch fed by streamed H2D chunks, "
                  "chunk-gated D2H)",
            False: "ts_hasf_batch_host (C ABI, pinned host buffers; chunked H2D / kernel / D2H pipeline)"}
PAPER_CPU_IMG_S = 32.0   # PAPER.md:13,330 (2x Xeon E5405, unknown r / images): context only


def bytes_per_image(cfg) -> int:
    """SURVEY §8(d) contract: 8 stages per radius x 4 B/px."""
    return 32 * cfg.r_max * cfg.h * cfg.w


def peak_hbm():
    path = os.path.join(REPO, "MEASURED_PEAKS.json")
    try:
        with open(path) as fh:
            return float(json.load(fh)["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs)"
    except Exception:
        return 6650.0, "fallback (B200_PROFILING.md)"


def traffic_from_profiles(cfg_name):
    path = os.path.join(REPO, "profiles", "ncu_traffic.json")
    try:
        with open(path) as fh:
            return json.load(fh).get(cfg_name)
    except Exception:
        return None


class ClockSampler:
    """SM clocks and clock-event (throttle) reasons sampled through NVML every
    ~2 ms on a background thread; mark(True/False) brackets the timed region
    and summary() reports the samples taken inside it (falls back to
    nvidia-smi -lms 10 when NVML is unavailable)."""

    REASONS = (("hw_slowdown", "nvmlClocksEventReasonHwSlowdown"),
               ("hw_thermal_slowdown", "nvmlClocksEventReasonHwThermalSlowdown"),
               ("sw_thermal_slowdown", "nvmlClocksEventReasonSwThermalSlowdown"),
               ("sw_power_cap", "nvmlClocksEventReasonSwPowerCap"),
               ("hw_power_brake", "nvmlClocksEventReasonHwPowerBrakeSlowdown"))

    def __init__(self, index=0):
        self.index = index
        self.samples = []        # (in_timed_region, sm_mhz, reasons)
        self.max_mhz = None
        self.inside = False
        self.stop = threading.Event()
        self.t = None
        self.source = None

    def __enter__(self):
        try:
            import pynvml as N
            N.nvmlInit()
            h = N.nvmlDeviceGetHandleByIndex(self.index)
            self.max_mhz = float(N.nvmlDeviceGetMaxClockInfo(h, N.NVML_CLOCK_SM))
            bits = [(nm, getattr(N, attr)) for nm, attr in self.REASONS if hasattr(N, attr)]

            def run():
                while not self.stop.is_set():
                    try:
                        mhz = float(N.nvmlDeviceGetClockInfo(h, N.NVML_CLOCK_SM))
                        r = int(N.nvmlDeviceGetCurrentClocksEventReasons(h))
                        self.samples.append((self.inside, mhz, [nm for nm, b in bits if r & b]))
                    except Exception:
                        pass
                    time.sleep(0.002)
            self.source = "nvml (2 ms)"
        except Exception:
            run = self._smi
            self.source = "nvidia-smi -lms 10"
        self.t = threading.Thread(target=run, daemon=True)
        self.t.start()
        time.sleep(0.05)
        return self

    def _smi(self):
        q = ("clocks.sm,clocks.max.sm,clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
             "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")
        try:
            proc = subprocess.Popen(["nvidia-smi", "-i", str(self.index), f"--query-gpu={q}",
                                     "--format=csv,noheader,nounits", "-lms", "10"],
                                    stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
        except Exception:
            return
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for line in proc.stdout:
            if self.stop.is_set():
                break
            parts = [x.strip() for x in line.split(",")]
            try:
                mhz, self.max_mhz = float(parts[0]), float(parts[1])
            except (ValueError, IndexError):
                continue
            self.samples.append((self.inside, mhz, [nm for nm, v in zip(names, parts[2:6])
                                                    if v.lower().startswith("active")]))
        proc.terminate()

    def mark(self, inside):
        self.inside = inside

    def __exit__(self, *a):
        self.stop.set()
        if self.t:
            self.t.join(timeout=5)

    def summary(self):
        inside = [s for s in self.samples if s[0]]
        sm = [s[1] for s in inside]
        reasons = sorted({r for s in inside for r in s[2]})
        return {"sm_mhz": float(np.median(sm)) if sm else None, "sm_max_mhz": self.max_mhz,
                "reasons": reasons, "samples": len(sm), "source": self.source}


def dist_env():
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return world, rank, local


def cpu_reference(cfg, images, threads):
    import oracle as O
    keep = avoid = None
    if cfg.constraints > 0:
        keep, avoid = W.constraint_masks(cfg, images)
    t0 = time.perf_counter()
    O.hasf_batch(images, cfg.r_max, cfg.fg, keep=keep, avoid=avoid, threads=threads)
    return time.perf_counter() - t0


def cpu_sample(cfg, cores, imgs=None):
    """Bounded CPU sample of the workload: (batch, images_equivalent, description).
    Images up to 2048^2: whole images (2 per core for <= 512^2, 1 per core
    otherwise).  Larger (c3, 8192^2): the image cut into 2048^2 tiles, each
    smoothed as an independent HASF -- the same pixel work, not the same output."""
    if cfg.h * cfg.w <= 2048 * 2048:
        k = max(1, min(cfg.n, cores * 2 if cfg.h * cfg.w <= 512 * 512 else cores))
        batch = imgs[:k] if imgs is not None and len(imgs) >= k else W.config_batch(cfg, 0, k)
        return batch, float(k), f"{k} images of {cfg.name} ({cfg.h}x{cfg.w}, r_max={cfg.r_max})"
    img = imgs[0] if imgs is not None else W.config_image(cfg, 0)
    t = 2048
    tiles = np.stack([img[y:y + t, x:x + t] for y in range(0, cfg.h, t) for x in range(0, cfg.w, t)])
    return tiles, len(tiles) * t * t / float(cfg.h * cfg.w), \
        f"{len(tiles)} independent {t}x{t} tiles covering one {cfg.name} image (r_max={cfg.r_max}; work-equivalent)"


# ---- reference arm: the stock reference package on the host cores --------
_REF = None


def _ref_init(path):
    """Pool worker: import the unmodified reference and JIT its numba kernels."""
    global _REF
    sys.path.insert(0, path)
    import toposmooth
    _REF = toposmooth
    z = np.zeros((16, 16), np.uint8)
    z[4:12, 4:12] = 1
    toposmooth.hasf(z, toposmooth.SmoothingConfig(r_max=2, adj=toposmooth.ADJ_84))
    toposmooth.hasf(z, toposmooth.SmoothingConfig(r_max=2, adj=toposmooth.ADJ_48))


def _ref_one(job):
    img, r_max, fg, keep, avoid = job
    adj = _REF.ADJ_84 if fg == 8 else _REF.ADJ_48
    # reference smoothing.py:187-212, one worker per process
    return _REF.hasf(img, _REF.SmoothingConfig(r_max=r_max, adj=adj, keep=keep, avoid=avoid, workers=1))


def stock_reference_available():
    if not os.path.isdir(os.path.join(REF_DIR, "toposmooth")):
        return False, "baseline/_ref not installed"
    try:
        import numba  # noqa: F401
        import scipy  # noqa: F401
    except Exception as e:  # pragma: no cover
        return False, f"reference dependency missing: {e}"
    return True, ""


def ref_sample_count(cfg, cores):
    """Images per timed step: a bounded sample (~1 s of the whole host)."""
    px = cfg.h * cfg.w
    if px <= 256 * 256:
        return min(cfg.n, 8 * cores)
    if px <= 512 * 512:
        return min(cfg.n, 2 * cores)
    return min(cfg.n, cores)


def physical_cores():
    pairs, phys, core = set(), None, None
    try:
        with open("/proc/cpuinfo") as fh:
            for line in fh:
                if line.startswith("physical id"):
                    phys = line.split(":")[1].strip()
                elif line.startswith("core id"):
                    core = line.split(":")[1].strip()
                elif not line.strip():
                    if phys is not None and core is not None:
                        pairs.add((phys, core))
                    phys = core = None
    except OSError:
        return None
    if phys is not None and core is not None:
        pairs.add((phys, core))
    return len(pairs) or None


def repo_libs_mapped():
    """In-repo shared objects mapped into this process (evidence for the arm's
    provenance: the reference arm must map none of the product's)."""
    libs = set()
    try:
        with open("/proc/self/maps") as fh:
            for ln in fh:
                path = ln.split()[-1] if len(ln.split()) >= 6 else ""
                if path.endswith(".so") and os.path.realpath(path).startswith(os.path.realpath(REPO)):
                    libs.add(os.path.relpath(os.path.realpath(path), os.path.realpath(REPO)))
    except OSError:
        pass
    return sorted(libs)


def run_reference(args, cfg):
    """--impl reference: the reference's own CPU implementation on this box's
    host cores.  Preferred: the UNMODIFIED toposmooth package (numba) from
    baseline/_ref as a process pool of os.cpu_count() workers, each running
    hasf(workers=1) on whole images (the reference's
    fair multicore throughput: its engine holds the GIL).  Fallback: the
    oracle's C restatement on all host threads.  The port is timed beside it
    and checked bit-exact against the stock reference's outputs."""
    world, rank, _ = dist_env()
    if rank != 0:
        return 0
    cores = os.cpu_count() or 1
    k = ref_sample_count(cfg, cores)
    if cfg.h * cfg.w > 2048 * 2048:
        imgs, equiv, desc = cpu_sample(cfg, cores)
    else:
        imgs, equiv = W.config_batch(cfg, 0, k), float(k)
        desc = f"{k} images of {cfg.name} ({cfg.h}x{cfg.w}, r_max={cfg.r_max})"
    ok, why = stock_reference_available()
    line_extra = {}
    if ok:
        import multiprocessing as mp
        ks = avs = [None] * len(imgs)
        if cfg.constraints > 0:
            ks, avs = W.constraint_masks(cfg, imgs)
        jobs = [(im, cfg.r_max, cfg.fg, k_, a_) for im, k_, a_ in zip(imgs, ks, avs)]
        with mp.get_context("fork").Pool(cores, initializer=_ref_init, initargs=(REF_DIR,)) as pool:
            outs = None
            for _ in range(args.warmup):
                outs = pool.map(_ref_one, jobs, chunksize=1)
            t = 0.0
            for _ in range(args.steps):
                t0 = time.perf_counter()
                outs = pool.map(_ref_one, jobs, chunksize=1)
                t += time.perf_counter() - t0
        value = args.steps * equiv / t
        # the port beside it (not the arm's value): same sample, all host threads
        import oracle as O
        tp = cpu_reference(cfg, imgs, cores)
        port_out = O.hasf_batch(imgs, cfg.r_max, cfg.fg, keep=None if cfg.constraints <= 0 else ks,
                                avoid=None if cfg.constraints <= 0 else avs, threads=cores)
        same = outs is not None and all(np.array_equal(a, b) for a, b in zip(outs, port_out))
        kind = "reference"
        sample = (f"{desc} per step; unmodified toposmooth 0.1.0 (numba) from baseline/_ref, hasf(workers=1) "
                  f"in a pool of {cores} processes (BASELINE.md §2 (iii)); warm-up steps JIT every worker")
        line_extra = {"port": {"value": equiv / tp, "unit": "images/s", "cores": cores,
                               "sample": f"{desc}, oracle/ C restatement on {cores} threads",
                               "bit_exact_vs_stock_reference": bool(same)}}
    else:
        for _ in range(args.warmup):
            cpu_reference(cfg, imgs[:1], 1)
        t = 0.0
        for _ in range(args.steps):
            t += cpu_reference(cfg, imgs, cores)
        value = args.steps * equiv / t
        kind = "port"
        sample = (f"{desc} per step, oracle/ C restatement of the reference (hasf, smoothing.py:187-212) "
                  f"on {cores} host threads ({why})")
    line = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": "images/s", "n_gpus": args.gpus,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1e3 * t / args.steps,
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "u8",
        "data": "synthetic (SURVEY §8d generator, per-image seeds)",
        "config": {"workload": f"{cfg.name}: {cfg.n}x{cfg.h}x{cfg.w} per GPU, r_max={cfg.r_max}, "
                               f"({cfg.fg},{12 - cfg.fg})", "sample_images_per_step": equiv,
                   "same_config_note": "each step times a bounded sample of the workload's images "
                                       "(BASELINE.md §2 subsampling); images/s is per-image throughput"},
        "cpu_baseline": {"value": value, "unit": "images/s", "cores": cores, "kind": kind, "sample": sample,
                         "physical_cores": physical_cores(), "logical_cpus": os.cpu_count()},
        "e2e": {"value": value, "unit": "images/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
        **line_extra,
        "repo_libs_mapped": repo_libs_mapped(),
    }
    print(json.dumps(line), flush=True)
    return 0


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--config", default="c1", choices=sorted(W.CONFIGS))
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--batch", type=int, default=0, help="override images per rank")
    ap.add_argument("--smem-budget", type=int, default=-1)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--e2e-steps", type=int, default=0, help="default: = steps")
    ap.add_argument("--verify", type=int, default=2, help="images checked bit-exact vs the oracle")
    ap.add_argument("--cluster-teams", type=int, default=1,
                    help="teams of 2..8 CTAs (large images) as thread-block clusters (1) or cooperative launches (0)")
    ap.add_argument("--host-streaming", type=int, default=1,
                    help="e2e host entry: 1 = one launch fed by streamed chunks, 0 = chunked launches")
    args = ap.parse_args()
    cfg = W.CONFIGS[args.config]
    if args.batch > 0:
        cfg = W.Config(**{**cfg.__dict__, "n": args.batch})
    if args.warmup < 3 and args.impl == "ours":
        print("warning: warmup < 3 violates the timing rules", file=sys.stderr)
    if args.impl == "reference":
        return run_reference(args, cfg)

    import torch
    import torch.distributed as dist

    import paper_1603_09337_b200 as P
    from paper_1603_09337_b200 import _lib
    from paper_1603_09337_b200.dist import max_over_ranks

    world, rank, local = dist_env()
    torch.cuda.set_device(local)
    # a rendezvous is set up (torchrun, any N): the barriers and the max-over-ranks reduce go through NCCL
    grouped = world > 1 or ("RANK" in os.environ and "MASTER_ADDR" in os.environ)
    if grouped:
        dist.init_process_group("nccl", init_method="env://", device_id=torch.device("cuda", local))
    if args.smem_budget >= 0:
        _lib.load().ts_set_smem_budget(args.smem_budget)
    _lib.load().ts_set_cluster_teams(args.cluster_teams)
    adj = P.ADJ_84 if cfg.fg == 8 else P.ADJ_48

    # this rank's images: indices rank*n .. rank*n + n - 1 (distinct seeds, weak scaling)
    imgs_np = W.config_batch(cfg, rank * cfg.n, cfg.n)
    x = torch.from_numpy(imgs_np).cuda()
    out = torch.empty_like(x)
    # constrained configs (c1k): seeded keep / avoid control images, resident too
    keep_np = avoid_np = None
    if cfg.constraints > 0:
        keep_np, avoid_np = W.constraint_masks(cfg, imgs_np, rank * cfg.n)
    kd = None if keep_np is None else torch.from_numpy(keep_np).cuda()
    ad = None if avoid_np is None else torch.from_numpy(avoid_np).cuda()
    kp = None if kd is None else kd.data_ptr()
    ap_ = None if ad is None else ad.data_ptr()
    stream = torch.cuda.current_stream()
    lib = _lib.load()

    def step():
        _lib.check(lib.ts_hasf_batch(x.data_ptr(), out.data_ptr(), cfg.n, cfg.h, cfg.w, cfg.r_max, cfg.fg,
                                     kp, ap_, stream.cuda_stream, None))

    flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")   # > 126 MB L2

    for _ in range(args.warmup):
        step()
    torch.cuda.synchronize()
    if grouped:
        dist.barrier()

    starts = [torch.cuda.Event(enable_timing=True) for _ in range(args.steps)]
    ends = [torch.cuda.Event(enable_timing=True) for _ in range(args.steps)]
    with ClockSampler(local) as clk:
        torch.cuda.synchronize()
        if grouped:
            dist.barrier()
        clk.mark(True)
        for i in range(args.steps):
            flush.fill_(i & 0xFF)          # evict L2 between timed steps (not timed)
            starts[i].record(stream)
            step()
            ends[i].record(stream)
        torch.cuda.synchronize()
        clk.mark(False)
        if grouped:
            dist.barrier()
    step_ms = [s.elapsed_time(e) for s, e in zip(starts, ends)]
    t_ms = max_over_ranks(float(sum(step_ms)))
    total_images = cfg.n * world * args.steps
    value = total_images / (t_ms / 1e3)

    # stats + correctness (outside the timed region): topology invariants of
    # every output (device component counts), bit-exactness on a sample
    _, stats = P.hasf_batch(x, cfg.r_max, adj, keep=kd, avoid=ad, stats=True)
    fi, bi = P.topology_counts(x, adj)
    fo, bo = P.topology_counts(out, adj)
    topo_ok = int(np.sum((fi == fo) & (bi == bo)))
    assert topo_ok == cfg.n, f"topology changed on {cfg.n - topo_ok} images"
    topo_summary = {"images": cfg.n, "preserved": topo_ok,
                    "fg_components_mean": float(fi.mean()), "bg_components_mean": float(bi.mean())}
    verified = 0
    if args.verify > 0 and rank == 0 and cfg.h * cfg.w <= 2048 * 2048:
        import oracle as O
        k = min(args.verify, cfg.n, 1 if cfg.h * cfg.w > 512 * 512 else args.verify)
        want = O.hasf_batch(imgs_np[:k], cfg.r_max, cfg.fg, keep=None if keep_np is None else keep_np[:k],
                            avoid=None if avoid_np is None else avoid_np[:k])
        got = out[:k].cpu().numpy()
        assert np.array_equal(got, want), "bench output differs from the oracle"
        if keep_np is not None:   # the constraints held on every output
            o = out.cpu().numpy()
            assert np.all(o[keep_np == 1] == 1) and np.all(o[avoid_np == 1] == 0)
        verified = k

    # e2e through the C ABI host-buffer entry, pinned host memory
    e2e_steps = args.e2e_steps or args.steps
    lib.ts_set_host_streaming(args.host_streaming)
    hin = torch.from_numpy(imgs_np).pin_memory()
    hout = torch.empty_like(hin).pin_memory()
    hk = None if keep_np is None else torch.from_numpy(keep_np).pin_memory()
    ha = None if avoid_np is None else torch.from_numpy(avoid_np).pin_memory()
    hkp = None if hk is None else hk.data_ptr()
    hap = None if ha is None else ha.data_ptr()

    def e2e_step():
        _lib.check(lib.ts_hasf_batch_host(hin.data_ptr(), hout.data_ptr(), cfg.n, cfg.h, cfg.w, cfg.r_max,
                                          cfg.fg, hkp, hap, stream.cuda_stream))

    e2e_step()
    torch.cuda.synchronize()
    if grouped:
        dist.barrier()
    t0 = time.perf_counter()
    e_start = torch.cuda.Event(enable_timing=True)
    e_end = torch.cuda.Event(enable_timing=True)
    e_start.record(stream)
    for _ in range(e2e_steps):
        e2e_step()
    e_end.record(stream)
    torch.cuda.synchronize()
    e2e_ms = max_over_ranks(e_start.elapsed_time(e_end))
    wall_ms = (time.perf_counter() - t0) * 1e3
    assert np.array_equal(hout.numpy(), out.cpu().numpy())
    e2e_value = cfg.n * world * e2e_steps / (e2e_ms / 1e3)
    # bytes that actually cross the host link per step (ts_hasf_batch_host):
    # the default streamed entry bit-packs the image and any keep / avoid
    # planes on the host (32 px per uint32 word), team-sized images (> 1024^2)
    # too unless TS_STREAM_BIG=0; otherwise uint8 planes
    packed = args.host_streaming == 1 and (cfg.h * cfg.w <= 1024 * 1024 or os.environ.get("TS_STREAM_BIG", "1") != "0")
    planes = 1 + (keep_np is not None) + (avoid_np is not None)   # inputs: image + control images
    link_in = planes * (cfg.n * cfg.h * ((cfg.w + 31) // 32) * 4 if packed else cfg.n * cfg.h * cfg.w)
    link_bytes = cfg.n * cfg.h * ((cfg.w + 31) // 32) * 4 if packed else cfg.n * cfg.h * cfg.w
    link_fmt = "bit-packed rows (uint32, 32 px/word)" if packed else "uint8 planes"

    if rank == 0:
        peak, peak_src = peak_hbm()
        bpi = bytes_per_image(cfg)
        kernel_s = t_ms / 1e3 / args.steps          # one fused launch per step
        achieved = bpi * cfg.n / kernel_s / 1e9
        cpu = None
        if not args.no_cpu_baseline and world >= 1:
            cores = os.cpu_count() or 1
            sample, equiv, desc = cpu_sample(cfg, cores, imgs_np)
            ts_ = cpu_reference(cfg, sample, cores)
            cpu = {"value": equiv / ts_, "unit": "images/s", "cores": cores, "kind": "port",
                   "sample": f"{desc}, oracle/ C restatement of the reference hasf on {cores} host "
                             f"threads, {ts_:.1f} s"}
        plan = np.zeros(6, np.int64)
        lib.ts_hasf_plan(cfg.h, cfg.w, cfg.r_max, int(keep_np is not None), int(avoid_np is not None),
                         plan.ctypes.data)
        line = {
            "metric": METRIC, "value": value, "unit": "images/s", "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": t_ms / args.steps, "higher_is_better": True,
            "scaling": "weak", "vs_baseline": None, "dtype": "u8",
            "data": "synthetic (SURVEY §8d generator, per-image seeds; paper images not shipped)",
            "config": {"workload": f"{cfg.name}: {cfg.n}x{cfg.h}x{cfg.w} per GPU, r_max={cfg.r_max}, "
                                   f"({cfg.fg},{12 - cfg.fg})", "global_batch": cfg.n * world,
                       "image": [cfg.h, cfg.w], "r_max": cfg.r_max, "adjacency": [cfg.fg, 12 - cfg.fg],
                       "constraints": (None if cfg.constraints <= 0 else
                                       f"seeded keep / avoid control images, {cfg.constraints:.0%} of object / "
                                       f"background pixels (W.constraint_masks)"),
                       "parallelism": f"images sharded over {world} GPU(s), no collective",
                       "l2": "flushed between timed steps (256 MiB fill, not timed); per-step CUDA events",
                       "scheduler": ("library defaults: (segment, image) tasks for batches above one wave; the fine "
                                     "tail (1 or 2 one-stage segments) chosen by the library from its first three "
                                     "launches, i.e. inside the warm-up" if not os.environ.get("TS_SEG_FINE") and
                                     os.environ.get("TS_SEG_TUNE", "1") != "0" else "fine tail fixed by environment"),
                       "plan": {"ctas_per_wave": int(plan[0]), "ctas_per_sm": int(plan[1]),
                                "smem_bytes": int(plan[2]), "smem_mask": int(plan[3]),
                                "gws_bytes_per_cta": int(plan[4]), "threads_per_cta": int(plan[5])}},
            "mpix_per_s": value * cfg.h * cfg.w / 1e6,
            "roofline": {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s",
                         "frac": achieved / peak, "traffic": traffic_from_profiles(cfg.name),
                         "peak_source": peak_src,
                         "algorithmic_bytes_per_launch": bpi * cfg.n,
                         "bytes_model": "32*r_max*H*W per image (SURVEY §8d: 8 stages/radius x 4 B/px)",
                         "kernel": "ts::hasf_kernel (one launch per step)"},
            "e2e": {"value": e2e_value, "unit": "images/s", "h2d_bytes_per_step": link_in,
                    "d2h_bytes_per_step": link_bytes, "wall_ms": wall_ms,
                    "host_uint8_bytes_per_step": {"read": planes * cfg.n * cfg.h * cfg.w,
                                                  "written": cfg.n * cfg.h * cfg.w},
                    "link_format": link_fmt, "path": E2E_PATH[args.host_streaming != 0]},
            "gpu_launches": args.steps,
            "cpu_baseline": cpu,
            "clocks": clk.summary(),
            "engine_stats_per_image": {"sweeps": float(stats[:, 0].mean()), "fixpoint_passes": float(stats[:, 1].mean()),
                                       "engine_calls": float(stats[:, 2].mean()), "flips": float(stats[:, 3].mean())},
            "verified_images_vs_oracle": verified,
            "topology_verified": topo_summary,
            "step_ms": step_ms,
            "paper_cpu_context_img_s": PAPER_CPU_IMG_S,
            "repo_libs_mapped": repo_libs_mapped(),
        }
        print(json.dumps(line), flush=True)
    if grouped:
        dist.destroy_process_group()
    return 0


if __name__ == "__main__":
    sys.exit(main())
