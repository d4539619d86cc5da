#!/bin/bash
for r in 1 2; do for lib in ab/*.so; do echo -n "$lib: "; DCOMP_LIB=$lib python tools/profile_crc.py 384 2>&1 | tail -1; done; done
