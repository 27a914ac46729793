"""Shared-memory bank conflicts per source function / line from an ncu source page CSV
(`--page source --print-source cuda,sass --csv`, tools/ncu_raw.sh): excessive wavefronts
(= wavefronts - ideal) of every shared-memory instruction.
    python tools/ncu_conflicts.py gpurun_out/srcs_c1.csv"""
import csv
import os
import re
import sys
from collections import defaultdict

csv.field_size_limit(10**9)
here = os.path.dirname(os.path.abspath(__file__))
src = open(os.path.join(here, "..", "paper_1603_09337_b200", "csrc", "ts_hasf_impl.cuh")).read().split("\n")
regions = []
for i, l in enumerate(src, 1):
    m = re.match(r'^(?:static\s+)?(?:template <[^>]*>\s*)?(?:static\s+)?(?:__device__|__global__)[^(]*?(\w+)\s*\(', l)
    if m:
        regions.append((i, m.group(1)))


def region(line):
    name = "?"
    for s, n in regions:
        if s <= line:
            name = n
    return name


hdr = None
cur_file = cur_line = None
seen = set()
agg = defaultdict(lambda: [0, 0, 0])
lines = defaultdict(lambda: [0, 0, 0])
for r in csv.reader(open(sys.argv[1])):
    if not r:
        continue
    if r[0] == "File Path":
        cur_file = r[1].split("/")[-1]
        continue
    if r[0] == "Function Name":
        continue
    if r[0] == "Line No":
        hdr = r
        ix = {h: i for i, h in enumerate(hdr)}
        continue
    if hdr is None or len(r) != len(hdr):
        continue
    if r[0]:
        cur_line = int(r[0])
        continue
    if not r[2].startswith("0x") or r[2] in seen:
        continue
    seen.add(r[2])

    def g(k):
        x = r[ix[k]]
        return int(float(x)) if x not in ("", "-") else 0

    v = (g("L1 Wavefronts Shared Excessive"), g("L1 Wavefronts Shared"), g("L1 Wavefronts Shared Ideal"))
    reg = region(cur_line) if cur_file == "ts_hasf_impl.cuh" else cur_file
    for i in range(3):
        agg[reg][i] += v[i]
        lines[(cur_file, cur_line)][i] += v[i]
tot = [sum(a[i] for a in agg.values()) for i in range(3)]
print("shared-memory wavefronts %d, ideal %d, excessive (bank conflicts) %d = %.1f%%" % (tot[1], tot[2], tot[0], 100.0 * tot[0] / max(1, tot[1])))
print("%-22s %10s %12s %10s" % ("function", "excess", "wavefronts", "excess/wf"))
for reg, a in sorted(agg.items(), key=lambda kv: -kv[1][0])[:16]:
    print("%-22s %9.1f%% %11.1f%% %10.2f" % (reg[:22], 100.0 * a[0] / max(1, tot[0]), 100.0 * a[1] / max(1, tot[1]), a[0] / max(1, a[1])))
print("\nlines (ts_hasf_impl.cuh of the profiled build):")
for (f, ln), b in sorted(lines.items(), key=lambda kv: -kv[1][0])[:14]:
    t = src[ln - 1].strip()[:90] if f == "ts_hasf_impl.cuh" and ln <= len(src) else f
    print("%6d excess %5.1f%%  wavefronts %5.1f%%  %s" % (ln, 100.0 * b[0] / max(1, tot[0]), 100.0 * b[1] / max(1, tot[1]), t))
