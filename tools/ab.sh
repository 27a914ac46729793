#!/bin/bash
# A/B driver on the GPU box: tools/ab.sh "<prof args>" lib1 lib2 ...  (lib "cur" = in-tree build)
args="$1"; shift
for lib in "$@"; do
  if [ "$lib" = cur ]; then unset TS_LIB_PATH; else export TS_LIB_PATH=$PWD/alt/$lib.so; fi
  echo "== $lib $args"
  python tools/prof_hasf.py $args
done
