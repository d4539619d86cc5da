#!/bin/bash
# A/B the resident decode across library builds in ab/*.so (interleaved runs).
for r in 1 2; do
  for lib in ab/*.so; do
    echo -n "$lib: "; DCOMP_LIB=$lib python tools/profile_decode.py --layers 24 --iters 8 2>&1 | grep "iter 7"
  done
done
