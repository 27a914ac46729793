#!/bin/bash
# same-box A/B of library builds: tools/exp_ab.sh "<prof_hasf args>" lib...   ("cur" = in-tree)
args="$1"; shift
for lib in "$@"; do
  if [ "$lib" = cur ]; then unset TS_LIB_PATH; else export TS_LIB_PATH=$PWD/alt/$lib.so; fi
  echo -n "$lib [$args]: "
  python tools/prof_hasf.py $args --repeat 4 --stats 0 | python -c "import json,sys; d=json.load(sys.stdin); print('%.3f' % d['ms_min'], d.get('verify_bad',''))"
done
