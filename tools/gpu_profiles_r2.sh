#!/bin/bash
# Round-2 ncu summaries of the kernels whose numbers DESIGN.md quotes (one GPU).
set -x
mkdir -p gpurun_out/ncu
ncu --set full --import-source on -k regex:k_fused_ring -s 1 -c 1 -o gpurun_out/ncu/fused python tools/profile_fused.py 0 opt-6.7b > /dev/null 2>&1
python tools/ncu_summary.py gpurun_out/ncu/fused.ncu-rep > gpurun_out/ncu/r2_fused_ring.txt 2>&1
ncu --set full -k regex:k_crc_lanes -s 2 -c 1 -o gpurun_out/ncu/crc python tools/profile_crc.py 384 > /dev/null 2>&1
python tools/ncu_summary.py gpurun_out/ncu/crc.ncu-rep > gpurun_out/ncu/r2_crc_lanes_bench.txt 2>&1
ncu --set full -k regex:"k_colhist5|k_select4|k_apply5|k_prune_rowsw" -s 4 -c 4 -o gpurun_out/ncu/prune python tools/profile_prune.py > /dev/null 2>&1
python tools/ncu_summary.py gpurun_out/ncu/prune.ncu-rep > gpurun_out/ncu/r2_prune_kernels.txt 2>&1
ncu --set full -k regex:"k_quantize_v|k_absmax_v" -s 2 -c 6 -o gpurun_out/ncu/quant python tools/profile_quant.py > /dev/null 2>&1
python tools/ncu_summary.py gpurun_out/ncu/quant.ncu-rep > gpurun_out/ncu/r2_quantize_kernels.txt 2>&1
ls -la gpurun_out/ncu
