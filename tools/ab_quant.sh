#!/bin/bash
for lib in ab/*.so; do echo "== $lib"; DCOMP_LIB=$lib python tools/profile_quant.py 2>&1 | grep -E "quantize|absmax"; done
