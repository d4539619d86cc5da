#!/bin/bash
# wide vs narrow split-point decoder across chunk sizes (DCOMP_NARROW_MAX_CHUNK: 0 = wide only)
for cs in 65536 131072 262144 1048576 16777216; do
  for lim in 0 1073741824; do
    echo -n "chunk $cs narrow_lim $lim: "; DCOMP_NARROW_MAX_CHUNK=$lim python tools/profile_decode.py --model opt-2.7b --layers 8 --chunk-size $cs --iters 4 2>&1 | grep "iter 3"
  done
done
