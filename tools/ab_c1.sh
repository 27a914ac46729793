#!/bin/bash
# same-box A/B of c1 knobs: dense divisor, dense batch builds (alt/db*.so)
run() { python tools/prof_hasf.py --config ${CFG:-c1} --n 0 --repeat 6 --stats 0 "$@" | python -c "import json,sys; d=json.load(sys.stdin); v=sorted(d[k] for k in d if k.startswith('ms_') and k!='ms_min'); print('%.4f %.4f' % (v[0], v[1]))"; }
for dd in 4 2 3 6 8; do echo -n "dense_div $dd: "; run --dense-div $dd; done
for L in db1 db3; do echo -n "$L: "; TS_LIB_PATH=$PWD/alt/$L.so run; done
echo -n "cur again: "; run
