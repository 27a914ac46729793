#!/bin/bash
# GPU-box A/B: tools/ab_ms.sh "<prof args>" lib1 lib2 ...  -> one line per lib: kernel ms (min of the repeats), verify result
args="$1"; shift
for lib in "$@"; do
  if [ "$lib" = cur ]; then unset TS_LIB_PATH; else export TS_LIB_PATH=$PWD/alt/$lib.so; fi
  python tools/prof_hasf.py $args --stats 0 | python -c "import json,sys; d=json.load(sys.stdin); print('$lib', '$args', round(d['ms_min'],3), d.get('verify_bad',''))"
done
