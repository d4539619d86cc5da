#!/bin/bash
# A/B the GPU pack (encode chains) across ab/*.so builds
for r in 1 2; do for lib in ab/*.so; do echo -n "$lib: "; DCOMP_LIB=$lib python tools/time_pack.py opt-1.3b 2>&1 | tail -1; done; done
