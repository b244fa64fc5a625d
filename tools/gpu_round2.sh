#!/bin/bash
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_kernels_gpu.py -m gpu -x -q -k "tile or tcgen05" 2>&1 | tail -30 | tee gpurun_out/pytest_tc.txt
bash tools/gpu_tests.sh tests
timeout 900 python bench.py --steps 3 --warmup 2 --no-cpu-baseline --out gpurun_out/bench_phi.json > gpurun_out/bench_phi.log 2>&1
tail -c 2500 gpurun_out/bench_phi.log
bash tools/ncu_launches.sh
