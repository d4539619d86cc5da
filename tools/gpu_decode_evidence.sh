# Decode-kernel evidence only: bench line, launch list, ncu --set full of k_decode_segments, C3 sweep.
set -x
python bench.py > gpurun_out/bench.log 2>&1; echo "bench rc=$?"
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches.csv python bench.py --steps 2 --warmup 3 --no-cpu --e2e-steps 1 --no-tp-shard > gpurun_out/ncu_launch.log 2>&1; echo "launch rc=$?"
ncu --set full --import-source on --clock-control none -k regex:k_decode_segments -c 1 -o gpurun_out/decode_full python tools/profile_decode.py --layers 24 --iters 2 > gpurun_out/ncu_dec.log 2>&1; echo "ncu dec rc=$?"
python tools/sweeps.py chunks --sizes 16384,32768,65536,262144,1048576,4194304 --out gpurun_out/c3.json > gpurun_out/c3.log 2>&1; echo "c3 rc=$?"
