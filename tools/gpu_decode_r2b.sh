#!/bin/bash
# Bench line + ncu evidence for the decode kernel on the bench workload (one GPU).
set -x
mkdir -p gpurun_out/ncu
python bench.py > gpurun_out/bench_r2b.log 2>&1; echo "bench rc=$?"
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_r2b.csv python bench.py --steps 2 --warmup 3 --no-cpu --e2e-steps 1 > gpurun_out/ncu_launch.log 2>&1; echo "launch rc=$?"
ncu --set full --import-source on --clock-control none -k regex:k_decode_segments -c 1 -o gpurun_out/ncu/decode_r2b python bench.py --steps 2 --warmup 3 --no-cpu --e2e-steps 1 > gpurun_out/ncu_dec.log 2>&1; echo "full rc=$?"
python tools/ncu_summary.py gpurun_out/ncu/decode_r2b.ncu-rep > gpurun_out/ncu/r2_decode_bench_v2.txt 2>&1
python tools/ncu_traffic.py gpurun_out/ncu/decode_r2b.ncu-rep > gpurun_out/ncu/traffic_r2b.txt 2>&1
