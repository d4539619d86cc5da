#!/bin/bash
# A/B small-chunk decode (16 / 32 KiB chunks) across library builds in ab/*.so.
for cs in 16384 32768; do
  for lib in ab/*.so; do
    echo -n "$cs $lib: "; DCOMP_LIB=$lib python tools/profile_decode.py --model opt-2.7b --layers 8 --chunk-size $cs --iters 4 2>&1 | grep "iter 3"
  done
done
