#!/bin/bash
mkdir -p gpurun_out
bash tools/gpu_tests.sh tests
timeout 900 python bench.py --steps 3 --warmup 2 --out gpurun_out/bench_phi.json > gpurun_out/bench_phi.log 2>&1
tail -c 800 gpurun_out/bench_phi.log
timeout 1500 python tools/cap_sweep.py --caps 4,8,12,14,16 --tokens 32 --steps 2 --warmup 1 > gpurun_out/cap_sweep.log 2>&1
tail -6 gpurun_out/cap_sweep.log
timeout 600 python tools/replay_bench.py > gpurun_out/replay_bench.log 2>&1
tail -8 gpurun_out/replay_bench.log
