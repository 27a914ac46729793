#!/bin/bash
# GPU box: one ncu --set full capture of the fused kernel for a config, raw metric page as CSV
# (gpurun_out/raw_<cfg>.csv) -- for digging into memory-system counters.   tools/ncu_raw.sh c2 [extra prof args]
c=$1; shift
T=/tmp/ts_raw; mkdir -p $T gpurun_out
P="python tools/prof_hasf.py --config $c --n 0 --repeat 2 --stats 0 $*"
$P > $T/plain.log 2>&1 || { cat $T/plain.log; exit 1; }
ncu --set full --clock-control none --import-source on -k regex:hasf_kernel -s 1 -c 1 -o $T/full_$c -f $P > $T/ncu.log 2>&1
tail -2 $T/ncu.log
ncu -i $T/full_$c.ncu-rep --page raw --csv > gpurun_out/raw_$c.csv 2>/dev/null
ncu -i $T/full_$c.ncu-rep --page source --print-source cuda,sass --csv > gpurun_out/srcs_$c.csv 2>/dev/null
ls -la gpurun_out/raw_$c.csv gpurun_out/srcs_$c.csv
