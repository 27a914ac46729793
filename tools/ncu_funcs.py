"""Attribute an ncu SASS page to the kernel's noinline callees (address ranges
between CALL targets) and name each range by its dominant source region.
    python tools/ncu_funcs.py report.ncu-rep images"""
import csv
import re
import subprocess
import sys
import os
from collections import Counter

rep, nimg = sys.argv[1], float(sys.argv[2])
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


out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--print-source", "cuda,sass", "--csv"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(out.splitlines()))
hdr = None
cur_file = None
cur_line = None
ins = {}   # addr -> (samples, executed, srcregion)
calls = set()
for r in rows:
    if not r:
        continue
    if r[0] == "File Path":
        cur_file = r[1].split("/")[-1]
        continue
    if r[0] == "Function Name":
        continue
    if r[0] == "Line No":
        hdr = r
        continue
    if len(r) != len(hdr):
        continue
    if r[0]:
        cur_line = int(r[0])
        continue
    if not r[2].startswith("0x"):
        continue
    addr = int(r[2], 16)
    d = dict(zip(hdr, r))
    s = int(d["Warp Stall Sampling (All Samples)"] or 0)
    e = int(d["Instructions Executed"] or 0)
    reg = region(cur_line) if cur_file == "ts_hasf_impl.cuh" else cur_file
    a = ins.setdefault(addr, [0, 0, Counter(), r[3]])
    a[0] = max(a[0], s)
    a[1] = max(a[1], e)
    a[2][reg] += 1
    m = re.search(r"CALL\.REL\.NOINC\s+(0x[0-9a-f]+)", r[3])
    if m:
        calls.add(int(m.group(1), 16))
addrs = sorted(ins)
base = addrs[0]
starts = sorted({base} | {base + c for c in calls} | {c for c in calls if c > base})
starts = [s for s in starts if s in ins]
tot_s = sum(v[0] for v in ins.values())
tot_e = sum(v[1] for v in ins.values())
res = []
for i, st in enumerate(starts):
    en = starts[i + 1] if i + 1 < len(starts) else addrs[-1] + 1
    s = e = 0
    names = Counter()
    for a in addrs:
        if st <= a < en:
            s += ins[a][0]
            e += ins[a][1]
            names.update(ins[a][2])
    res.append((s, e, st - base, names.most_common(3)))
for s, e, off, nm in sorted(res, reverse=True)[:30]:
    print(f"+{off:#07x} samples {100 * s / tot_s:5.1f}%  instr {e / nimg / 1e6:5.2f}M/img  {nm}")

if len(sys.argv) > 3:
    # per-source-region breakdown inside one callee range (offset as printed)
    off = int(sys.argv[3], 16)
    st = base + off
    en = min([s for s in starts if s > st] + [addrs[-1] + 1])
    by = Counter()
    byi = Counter()
    for a in addrs:
        if st <= a < en:
            reg = ins[a][2].most_common(1)[0][0]
            by[reg] += ins[a][0]
            byi[reg] += ins[a][1]
    tot = sum(by.values())
    for k, v in by.most_common(25):
        print(f"   {k:24s} {100 * v / tot:5.1f}% of range  instr {byi[k] / nimg / 1e6:5.2f}M/img")
    if len(sys.argv) > 4:
        want = sys.argv[4]
        byl = Counter()
        # re-walk rows to get line numbers per address inside the range for the region
        cur_file = None
        cur_line = None
        for r in rows:
            if not r:
                continue
            if r[0] == "File Path":
                cur_file = r[1].split("/")[-1]
                continue
            if r[0] in ("Function Name", "Line No") or len(r) != len(hdr):
                continue
            if r[0]:
                cur_line = int(r[0])
                continue
            if not r[2].startswith("0x"):
                continue
            a = int(r[2], 16)
            if st <= a < en and cur_file == "ts_hasf_impl.cuh" and region(cur_line) == want:
                byl[cur_line] += int(dict(zip(hdr, r))["Warp Stall Sampling (All Samples)"] or 0)
        for ln, v in byl.most_common(12):
            print(f"      line {ln:5d} {100 * v / tot:5.1f}%  {src[ln - 1].strip()[:90]}")
