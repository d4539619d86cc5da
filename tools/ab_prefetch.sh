#!/bin/bash
# next-task L2 prefetch on/off (DCOMP_NO_PREFETCH=1 zeroes the task span bytes)
for r in 1 2; do
  for pf in 0 1; do
    echo -n "no_prefetch=$pf: "; DCOMP_NO_PREFETCH=$pf python tools/profile_decode.py --layers 24 --iters 8 2>&1 | grep "iter 7"
  done
done
