"""Aggregate an ncu source page (cuda,sass) by enclosing function of
ts_hasf_impl.cuh: warp-stall samples and executed instructions per region.
    python tools/ncu_regions.py report.ncu-rep [images]"""
import csv
import re
import subprocess
import sys
import os

rep = sys.argv[1]
nimg = float(sys.argv[2]) if len(sys.argv) > 2 else 1.0
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--print-source", "cuda,sass", "--csv"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(out.splitlines()))
here = os.path.dirname(os.path.abspath(__file__))
src = open(os.path.join(here, "..", "paper_1603_09337_b200", "csrc", "ts_hasf_impl.cuh")).read().split("\n")
regions = []
for i, l in enumerate(src, 1):
    m = re.match(r'^(?:template <[^>]*>\s*)?(?:__device__|__global__)[^(]*?(\w+)\s*\(', l)
    if m:
        regions.append((i, m.group(1)))


def region(line):
    name = "?"
    for s, n in regions:
        if s <= line:
            name = n
    return name


cur = hdr = None
agg = {}
stalls = {}
tot_s = tot_i = 0
for r in rows:
    if not r:
        continue
    if r[0] == "File Path":
        cur = r[1].split("/")[-1]
        continue
    if r[0] in ("Function Name",):
        continue
    if r[0] == "Line No":
        hdr = r
        continue
    if not r[0]:
        continue   # sass rows
    if len(r) != len(hdr):
        continue
    d = dict(zip(hdr, r))
    s = int(d["Warp Stall Sampling (All Samples)"] or 0)
    ins = int(d["Instructions Executed"] or 0)
    key = region(int(d["Line No"])) if cur == "ts_hasf_impl.cuh" else cur
    a = agg.setdefault(key, [0, 0])
    a[0] += s
    a[1] += ins
    st = stalls.setdefault(key, {})
    for k, v in d.items():
        if k.startswith("stall_") and "Not Issued" not in k and v not in ("", "-"):
            st[k[6:]] = st.get(k[6:], 0) + int(v)
    tot_s += s
    tot_i += ins
for k, (s, i) in sorted(agg.items(), key=lambda x: -x[1][0])[:25]:
    top = sorted(stalls[k].items(), key=lambda x: -x[1])[:4]
    tops = " ".join(f"{n}:{100 * v / max(1, s):.0f}" for n, v in top)
    print(f"{k:22s} samples {100 * s / tot_s:5.1f}%  instr {100 * i / tot_i:5.1f}% ({i / nimg / 1e6:.2f}M/img)  {tops}")
