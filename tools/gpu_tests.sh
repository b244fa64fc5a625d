#!/bin/bash
# usage: tools/gpu_tests.sh [pytest targets/args]; output under gpurun_out/
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/gpu.txt 2>&1
T="${@:-tests}"
timeout 1500 python -m pytest $T -m gpu -x -q 2>&1 | tail -80 | tee gpurun_out/pytest_gpu.txt
