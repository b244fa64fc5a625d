#!/bin/bash
# full GPU test suite + a short Phi bench
mkdir -p gpurun_out
bash tools/gpu_tests.sh tests
timeout 900 python bench.py --steps 3 --warmup 2 --no-cpu-baseline --out gpurun_out/bench_phi.json > gpurun_out/bench_phi.log 2>&1
tail -c 3000 gpurun_out/bench_phi.log
