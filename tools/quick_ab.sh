#!/bin/bash
# GPU-box quick check: kernel ms (min of 3) for the configs given (default c1 c4 c3 c2), then the gpu tests
for c in ${CONFIGS:-c1 c4 c3 c2}; do
  python tools/prof_hasf.py --config $c --n 0 --repeat 3 --stats 0 | python -c "import json,sys; d=json.load(sys.stdin); print('$c', round(d['ms_min'],3))"
done
[ "${TESTS:-1}" = 1 ] && python -m pytest tests -m gpu -x -q 2>&1 | tail -3
