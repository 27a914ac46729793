#!/bin/bash
# same-box A/B: alt/seg1.so (pre-segment build) vs the in-tree build at several segment settings
nvidia-smi --query-gpu=clocks.sm,clocks.max.sm --format=csv,noheader
for cfg in c1 c4; do
  echo "== $cfg alt/seg1"; TS_LIB_PATH=$PWD/alt/seg1.so python tools/prof_hasf.py --config $cfg --n 0 --repeat 6 --stats 0 | python -c "import json,sys; d=json.load(sys.stdin); print(sorted(d[k] for k in d if k.startswith('ms_') and k!='ms_min')[:4])"
  for combo in "0 0" "2 0" "4 4" "4 2" "4 0"; do set -- $combo
    echo "== $cfg cur seg=$1 fine=$2"; TS_SEG_STAGES=$1 TS_SEG_FINE=$2 python tools/prof_hasf.py --config $cfg --n 0 --repeat 6 --stats 0 | python -c "import json,sys; d=json.load(sys.stdin); print(sorted(d[k] for k in d if k.startswith('ms_') and k!='ms_min')[:4])"
  done
done
nvidia-smi --query-gpu=clocks.sm,clocks.max.sm --format=csv,noheader
