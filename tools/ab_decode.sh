#!/bin/bash
# A/B the resident decode across library builds in ab/*.so (interleaved runs).
# usage: tools/ab_decode.sh [model] [layers] [chunk_size]
M=${1:-opt-6.7b}; L=${2:-4}; C=${3:-16777216}
for r in 1 2 3; do
  for lib in ab/*.so; do
    echo -n "$lib: "; DCOMP_LIB=$lib python tools/profile_decode.py --model $M --layers $L --iters 8 --chunk-size $C 2>&1 | grep "iter 7"
  done
done
