#!/bin/bash
run() { python tools/prof_hasf.py --config $1 --n 0 --repeat 6 --stats 0 | python -c "import json,sys; d=json.load(sys.stdin); v=sorted(d[k] for k in d if k.startswith('ms_') and k!='ms_min'); print('%.4f %.4f' % (v[0], v[1]))"; }
for c in c1 c0; do for L in cur u4off cur u4off; do echo -n "$c $L: "; if [ $L = cur ]; then unset TS_LIB_PATH; else export TS_LIB_PATH=$PWD/alt/$L.so; fi; run $c; done; done
