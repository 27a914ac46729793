"""Summarise ncu captures into profiles/ (run in the build container).

    python tools/summarize_ncu.py --launches gpurun_out/launches_c1.csv \
        --full gpurun_out/full_c1.ncu-rep --tag r01_c1 --images 256 --bytes-per-image 41943040

Writes profiles/<tag>_launches.txt (per-kernel share of GPU time),
profiles/<tag>_full_summary.txt (key counters, stall mix, hottest source lines)
and updates profiles/ncu_traffic.json with the DRAM bytes of one launch.
"""
import argparse
import collections
import csv
import json
import os
import subprocess

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
SCALE = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "ns": 1e-3, "us": 1, "usecond": 1,
         "nsecond": 1e-3, "ms": 1e3, "msecond": 1e3}


def launches(path):
    rows = [r for r in csv.reader(open(path)) if r]
    hdr, data = None, []
    for r in rows:
        if r[0] == "ID":
            hdr = r
            continue
        if hdr and len(r) == len(hdr):
            data.append(dict(zip(hdr, r)))
    agg = collections.defaultdict(lambda: [0, 0.0])
    for d in data:
        if d.get("Metric Name") != "gpu__time_duration.sum":
            continue
        v = float(d["Metric Value"].replace(",", "")) * SCALE.get(d["Metric Unit"], 1)
        agg[d["Kernel Name"][:80]][0] += 1
        agg[d["Kernel Name"][:80]][1] += v
    tot = sum(v[1] for v in agg.values())
    lines = [f"{v[0]:5d} launches {v[1]:12.1f} us {100 * v[1] / tot:6.2f}%  {k}"
             for k, v in sorted(agg.items(), key=lambda kv: -kv[1][1])]
    return lines


def ncu_csv(rep, *args):
    return subprocess.run(["ncu", "-i", rep, *args, "--csv"], capture_output=True, text=True).stdout


def full(rep, images, bpi):
    raw = list(csv.reader(ncu_csv(rep, "--page", "raw").splitlines()))
    h, u, v = raw[0], raw[1], raw[2]
    d, un = dict(zip(h, v)), dict(zip(h, u))
    val = lambda k: float(d[k].replace(",", "")) * SCALE.get(un.get(k, ""), 1)  # noqa: E731
    keys = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
            "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "lts__throughput.avg.pct_of_peak_sustained_elapsed",
            "sm__throughput.avg.pct_of_peak_sustained_elapsed", "smsp__issue_active.avg.pct_of_peak_sustained_active",
            "sm__warps_active.avg.pct_of_peak_sustained_active", "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum",
            "l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum", "launch__registers_per_thread",
            "launch__shared_mem_per_block_dynamic", "launch__grid_size", "launch__block_size", "smsp__inst_executed.sum"]
    out = [f"{k:62s} {un.get(k, ''):>12s} {d.get(k)}" for k in keys if k in d]
    traffic = val("dram__bytes_read.sum") + val("dram__bytes_write.sum")
    out.append("")
    out.append(f"DRAM traffic per launch (read+write): {traffic:.4g} B = {traffic / images:.4g} B/image")
    if bpi:
        out.append(f"contract algorithmic bytes per launch: {bpi * images:.4g} B")
    stalls = [k for k in h if k.startswith("smsp__pcsamp_warps_issue_stalled") and not k.endswith("_not_issued")]
    tot = sum(float(d[k] or 0) for k in stalls) or 1.0
    out.append("\nwarp stall reasons (pc-sampling share):")
    for s, k in sorted(((float(d[k] or 0), k) for k in stalls), reverse=True)[:10]:
        out.append(f"  {k.replace('smsp__pcsamp_warps_issue_stalled_', ''):26s} {100 * s / tot:5.1f} %")
    src = list(csv.reader(ncu_csv(rep, "--page", "source", "--print-source", "cuda,sass").splitlines()))
    cur, samp, text = None, collections.Counter(), {}
    for r in src:
        if not r:
            continue
        if r[0] == "File Path":
            cur = r[1].split("/")[-1]
        elif r[0] and r[0].isdigit() and len(r) > 4:
            try:
                samp[(cur, int(r[0]))] += int(r[4])
                text[(cur, int(r[0]))] = r[1].strip()[:90]
            except ValueError:
                pass
    ts = sum(samp.values()) or 1
    out.append("\nhottest source lines (pc-sampling share):")
    for k, s in samp.most_common(15):
        out.append(f"  {100 * s / ts:5.1f}%  {k[0]}:{k[1]}  {text[k]}")
    return out, traffic


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--launches")
    ap.add_argument("--full")
    ap.add_argument("--tag", required=True)
    ap.add_argument("--images", type=int, default=256)
    ap.add_argument("--bytes-per-image", type=int, default=0)
    ap.add_argument("--config", default="c1")
    ap.add_argument("--cmd", default="")
    ap.add_argument("--out-dir", default=os.path.join(REPO, "profiles"),
                    help="where the summaries go (on the GPU box: a gpurun_out/ subdirectory)")
    a = ap.parse_args()
    prof = a.out_dir
    os.makedirs(prof, exist_ok=True)
    if a.launches:
        with open(os.path.join(prof, f"{a.tag}_launches.txt"), "w") as fh:
            fh.write(f"ncu --metrics gpu__time_duration.sum --clock-control none (cold-cache, serialised)\n{a.cmd}\n\n")
            fh.write("\n".join(launches(a.launches)) + "\n")
    if a.full:
        lines, traffic = full(a.full, a.images, a.bytes_per_image)
        with open(os.path.join(prof, f"{a.tag}_full_summary.txt"), "w") as fh:
            fh.write(f"ncu --set full --clock-control none --import-source on, one ts::hasf_kernel launch\n{a.cmd}\n\n")
            fh.write("\n".join(lines) + "\n")
        tj = os.path.join(prof, "ncu_traffic.json")
        data = json.load(open(tj)) if os.path.exists(tj) else {}
        data[a.config] = int(traffic)
        data[f"_{a.config}_source"] = f"profiles/{a.tag}_full_summary.txt"
        json.dump(data, open(tj, "w"), indent=1)


if __name__ == "__main__":
    main()
