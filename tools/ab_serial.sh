#!/bin/bash
# A/B the exact serial (index-less) decode across ab/*.so builds
for r in 1 2; do for lib in ab/*.so; do echo -n "$lib: "; DCOMP_LIB=$lib python tools/profile_serial.py 2 2>&1 | tail -1; done; done
