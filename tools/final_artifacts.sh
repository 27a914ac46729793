#!/bin/bash
# GPU-box script: everything the round's records are made of, on the current build --
# gpu tests, bench lines for every config (+ the reference arm), stress parity, host timeline of the
# e2e entry, per-config ncu launch lists and full-capture summaries (tools/profile_all.sh).
# Outputs under gpurun_out/final/ and gpurun_out/prof/.
set -u
O=gpurun_out/final; mkdir -p $O
python -m pytest tests -m gpu -q > $O/gpu_tests.log 2>&1; tail -1 $O/gpu_tests.log
for c in c1 c4 c2 c0 c3 c1k; do
  python bench.py --config $c > $O/bench_$c.json 2> $O/bench_$c.err; python tools/bench_summary.py $O/bench_$c.json
done
python bench.py --impl reference --steps 3 --warmup 3 > $O/bench_reference_c1.json 2> $O/bench_reference_c1.err
python tools/bench_summary.py $O/bench_reference_c1.json
TS_HOST_TRACE=1 python tools/e2e_trace.py > $O/e2e_host_timeline.txt 2>&1; tail -20 $O/e2e_host_timeline.txt | head -3
python tools/stress_parity.py --cases ${STRESS:-1500} --seed 9091 > $O/stress_parity.log 2>&1; tail -1 $O/stress_parity.log
./tools/probe/team_barrier_bin > $O/team_barrier_probe.txt 2>&1
./tools/probe/atomic_rate_bin > $O/atomic_rate_probe.txt 2>&1
TAG=r02 bash tools/profile_all.sh > $O/profile_all.log 2>&1; tail -3 $O/profile_all.log
