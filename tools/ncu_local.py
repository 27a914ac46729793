"""Per source function (of ts_hasf_impl.cuh) totals from an ncu source page CSV made with
`--page source --print-source cuda,sass --csv`: stall samples, executed instructions, local-memory
and global-memory L2 sectors -- where the spill traffic and the long-scoreboard stalls are.
    python tools/ncu_local.py gpurun_out/srcs_c2.csv [function-for-line-breakdown]"""
import csv
import os
import re
import sys
from collections import Counter, defaultdict

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


rows = csv.reader(open(sys.argv[1]))
want = sys.argv[2] if len(sys.argv) > 2 else None
hdr = None
cur_file = cur_line = None
K = ["Warp Stall Sampling (All Samples)", "Instructions Executed", "L2 Theoretical Sectors Local",
     "L2 Theoretical Sectors Global", "stall_long_sb", "stall_barrier"]
agg = defaultdict(lambda: [0] * len(K))
lines = defaultdict(lambda: [0] * len(K))
seen = set()
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
        ix = {h: i for i, h in enumerate(hdr)}
        continue
    if hdr is None or len(r) != len(hdr):
        continue
    if r[0]:
        cur_line = int(r[0])
        continue
    if not r[2].startswith("0x"):
        continue
    if r[2] in seen:      # an instruction is listed under every file that contributes to it
        continue
    seen.add(r[2])
    reg = region(cur_line) if cur_file == "ts_hasf_impl.cuh" else cur_file
    vals = []
    for k in K:
        x = r[ix[k]] if k in ix else "0"
        vals.append(int(float(x)) if x not in ("", "-") else 0)
    a = agg[reg]
    for i, v in enumerate(vals):
        a[i] += v
    if want and reg == want:
        b = lines[cur_line]
        for i, v in enumerate(vals):
            b[i] += v
tot = [sum(a[i] for a in agg.values()) for i in range(len(K))]
print("totals: samples %d  instr %.3g  local sectors %.3g  global sectors %.3g" % tuple(tot[:4]))
print("%-22s %8s %8s %8s %8s %8s %8s" % ("function", "samples", "instr", "local", "global", "long_sb", "barrier"))
for reg, a in sorted(agg.items(), key=lambda kv: -kv[1][0])[:28]:
    print("%-22s " % reg[:22] + " ".join("%7.1f%%" % (100.0 * a[i] / max(1, tot[i])) for i in range(len(K))))
if want:
    t = agg[want]
    print(f"\nlines of {want} (share of the function):")
    for ln, b in sorted(lines.items(), key=lambda kv: -kv[1][0])[:16]:
        print("  %5d " % ln + " ".join("%6.1f%%" % (100.0 * b[i] / max(1, t[i])) for i in range(len(K))) + "  " + src[ln - 1].strip()[:80])
