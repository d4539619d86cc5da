# One GPU session: bench line, C3/C4 sweeps, ncu captures of the two hot kernels.
set -x
python bench.py > gpurun_out/bench.log 2>&1; echo "bench rc=$?"
python tools/sweeps.py chunks --out gpurun_out/c3.json > gpurun_out/c3.log 2>&1; echo "c3 rc=$?"
python tools/sweeps.py partial --curve gpurun_out/c3.json --out gpurun_out/c4.json > gpurun_out/c4.log 2>&1; echo "c4 rc=$?"
ncu --set full --import-source on --clock-control none -k regex:k_decode_segments -c 1 -o gpurun_out/decode_full python tools/profile_decode.py --layers 24 --iters 2 > gpurun_out/ncu_dec.log 2>&1; echo "ncu dec rc=$?"
ITERS=2 ncu --set full --import-source on --clock-control none -k regex:k_fused_ring -s 1 -c 1 -o gpurun_out/fused_full python tools/profile_fused.py 0 > gpurun_out/ncu_fused.log 2>&1; echo "ncu fused rc=$?"
