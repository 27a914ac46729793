#!/bin/bash
# A/B of the segmented scheduler on the GPU box: bench lines per TS_SEG_STAGES value.
O=gpurun_out/seg; mkdir -p $O
for cfg in ${CFGS:-c1 c4}; do
  for s in ${SEGS:-0 2 4}; do
    TS_SEG_STAGES=$s python bench.py --config $cfg --steps 10 --warmup 3 --no-cpu-baseline --verify 2 > $O/${cfg}_s$s.json 2> $O/${cfg}_s$s.err
    python - "$O/${cfg}_s$s.json" "$cfg" "$s" <<'PY'
import json, sys
try:
    d = json.loads(open(sys.argv[1]).read().strip().splitlines()[-1])
    print(sys.argv[2], "seg", sys.argv[3], "ms/step %.3f" % d["ms_per_step"], "frac %.3f" % d["roofline"]["frac"],
          "e2e %.0f" % d["e2e"]["value"], "verified", d["verified_images_vs_oracle"])
except Exception as e:
    print(sys.argv[2], "seg", sys.argv[3], "FAILED", e)
PY
  done
done
