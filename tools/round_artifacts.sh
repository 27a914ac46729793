#!/bin/bash
# GPU-box script: tests, bench lines for every config, reference arm, ncu
# launch list + full capture of the c1 kernel.  Outputs under gpurun_out/art/.
set -u
O=gpurun_out/art; mkdir -p $O
python -m pytest tests -m gpu -q > $O/gpu_tests.log 2>&1; tail -2 $O/gpu_tests.log
for c in c1 c4 c2 c0 c3; do
  python bench.py --config $c > $O/bench_$c.json 2> $O/bench_$c.err; tail -c 300 $O/bench_$c.json
done
python bench.py --impl reference --steps 3 --warmup 3 > $O/bench_ref_c1.json 2> $O/bench_ref_c1.err; tail -c 400 $O/bench_ref_c1.json
CMD="python bench.py --steps 2 --warmup 3 --no-cpu-baseline --verify 0 --e2e-steps 1"
$CMD > $O/plain.log 2>&1 && ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/launches_c1.csv $CMD > $O/ncu_launch.log 2>&1
$CMD > $O/plain2.log 2>&1 && ncu --set full --clock-control none --import-source on -k regex:hasf_kernel -s 3 -c 1 -o $O/prof_c1 $CMD > $O/ncu_full.log 2>&1
tail -2 $O/ncu_full.log
