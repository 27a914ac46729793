#!/bin/bash
# GPU-box: per config, the launch list of the bench command and one ncu --set
# full capture of the fused kernel (prof_hasf: one launch over the whole
# config batch), summarised ON THE BOX into gpurun_out/prof/ (the .ncu-rep
# files are too large to bring back and are deleted).  CFGS overrides the list;
# TAG prefixes the summary names.
set -u
O=gpurun_out/prof; mkdir -p $O; T=/tmp/ts_prof; mkdir -p $T
TAG=${TAG:-r02}
declare -A IMGS=([c0]=1 [c1]=256 [c1k]=256 [c2]=32 [c3]=1 [c4]=1024)
declare -A BPI=([c0]=25165824 [c1]=41943040 [c1k]=41943040 [c2]=1342177280 [c3]=17179869184 [c4]=8388608)
for c in ${CFGS:-c1 c4 c2 c0 c1k c3}; do
  B="python bench.py --config $c --steps 2 --warmup 3 --no-cpu-baseline --verify 0 --e2e-steps 1"
  if [ "${LAUNCH:-1}" = 1 ]; then
    $B > $T/plain_$c.log 2>&1 && ncu --metrics gpu__time_duration.sum --clock-control none --csv \
        --log-file $T/launches_$c.csv $B > $T/ncu_launch_$c.log 2>&1
    python tools/summarize_ncu.py --launches $T/launches_$c.csv --tag ${TAG}_$c --config $c --out-dir $O --cmd "$B"
  fi
  P="python tools/prof_hasf.py --config $c --n 0 --repeat 2 --stats 0"
  $P > $T/prof_plain_$c.log 2>&1 && ncu --set full --clock-control none --import-source on -k regex:hasf_kernel \
      -s 1 -c 1 -o $T/full_$c -f $P > $T/ncu_full_$c.log 2>&1
  echo "$c: rc=$? $(tail -c 150 $T/ncu_full_$c.log | tr '\n' ' ')"
  python tools/summarize_ncu.py --full $T/full_$c.ncu-rep --tag ${TAG}_$c --config $c --images ${IMGS[$c]} \
      --bytes-per-image ${BPI[$c]} --out-dir $O --cmd "$P"
  cp $O/ncu_traffic.json $O/ncu_traffic_$c.json 2>/dev/null
  rm -f $T/full_$c.ncu-rep
done
