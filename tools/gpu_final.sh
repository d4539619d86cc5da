# Round-end evidence: tests, smoke, bench line, launch list of the bench command,
# ncu of the hot kernels, sweeps.
set -x
python -m pytest tests -x -q -m gpu > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?"
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?"
python bench.py > gpurun_out/bench.log 2>&1; echo "bench rc=$?"
python bench.py --impl reference --steps 5 --warmup 1 > gpurun_out/bench_ref.log 2>&1; echo "ref rc=$?"
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches.csv python bench.py --steps 2 --warmup 3 --no-cpu --e2e-steps 1 > gpurun_out/ncu_launch.log 2>&1; echo "launch rc=$?"
ncu --set full --import-source on --clock-control none -k regex:k_decode_segments -c 1 -o gpurun_out/decode_full python tools/profile_decode.py --layers 24 --iters 2 > gpurun_out/ncu_dec.log 2>&1; echo "ncu dec rc=$?"
ITERS=2 ncu --set full --import-source on --clock-control none -k regex:k_fused_ring -s 1 -c 1 -o gpurun_out/fused_full python tools/profile_fused.py 0 > gpurun_out/ncu_fused.log 2>&1; echo "ncu fused rc=$?"
python tools/sweeps.py chunks --sizes 16384,32768,65536,262144,1048576,4194304 --out gpurun_out/c3.json > gpurun_out/c3.log 2>&1; echo "c3 rc=$?"
python tools/sweeps.py partial --curve gpurun_out/c3.json --out gpurun_out/c4.json > gpurun_out/c4.log 2>&1; echo "c4 rc=$?"
python tools/int8_scaling.py --out gpurun_out/int8_scaling.json > gpurun_out/int8_scaling.log 2>&1; echo "int8 scaling rc=$?"
DCOMP_TIMELINE=1 python tools/e2e_timeline.py > gpurun_out/e2e_timeline.txt 2>&1; echo "timeline rc=$?"
