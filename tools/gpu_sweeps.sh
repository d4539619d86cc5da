set -x
ITERS=2 ncu --set full --import-source on --clock-control none -k regex:k_fused_ring -s 1 -c 1 -o gpurun_out/fused_v4 python tools/profile_fused.py 0 > gpurun_out/ncu_fused4.log 2>&1; echo "ncu rc=$?"
python tools/sweeps.py chunks --out gpurun_out/c3.json > gpurun_out/c3.log 2>&1; echo "c3 rc=$?"
python tools/sweeps.py partial --curve gpurun_out/c3.json --out gpurun_out/c4.json > gpurun_out/c4.log 2>&1; echo "c4 rc=$?"
