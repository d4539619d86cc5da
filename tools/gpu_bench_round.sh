set -x
python bench.py > gpurun_out/bench_v3.log 2>&1; echo "bench rc=$?"
tail -c 600 gpurun_out/bench_v3.log
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_v3.csv python bench.py --steps 2 --warmup 3 --no-cpu --e2e-steps 1 > gpurun_out/ncu_launch.log 2>&1; echo "launch rc=$?"
ncu --set full --import-source on --clock-control none -k regex:k_decode_segments -c 1 -o gpurun_out/bench_decode_v3 python bench.py --steps 2 --warmup 3 --no-cpu --e2e-steps 1 > gpurun_out/ncu_dec.log 2>&1; echo "full rc=$?"
