#!/bin/bash
# A/B the fused decode->GEMM across library builds in ab/*.so (interleaved runs).
for r in 1 2; do
  for lib in ab/*.so; do
    echo -n "$lib: "; DCOMP_LIB=$lib ITERS=6 python tools/profile_fused.py 0 2>&1 | grep "iter 5"
  done
done
