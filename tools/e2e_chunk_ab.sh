#!/bin/bash
# GPU-box A/B of the streamed host entry's chunk size (TS_CHUNK_BYTES), interleaved repeats
for rep in 1 2 3; do
for cb in ${CHUNKS:-4194304 2097152 3145728}; do
TS_CHUNK_BYTES=$cb tools/e2e_ab.sh 8:0 | sed "s/^/chunk $cb /"
done
done
