#!/bin/bash
# full round check on one B200: gpu tests, smoke, 1-GPU bench, replay bench
mkdir -p gpurun_out
bash tools/gpu_tests.sh tests
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.txt 2>&1; tail -3 gpurun_out/smoke.txt
timeout 900 python bench.py --steps 3 --warmup 3 --out gpurun_out/bench_phi.json > gpurun_out/bench_phi.log 2>&1
tail -c 1500 gpurun_out/bench_phi.log
timeout 600 python tools/replay_bench.py > gpurun_out/replay_bench.log 2>&1
tail -8 gpurun_out/replay_bench.log
