#!/bin/bash
mkdir -p gpurun_out
timeout 300 python bench.py --model tiny --steps 3 --warmup 1 --no-cpu-baseline > gpurun_out/bench_tiny.log 2>&1; echo "tiny rc=$?" >> gpurun_out/bench_tiny.log
timeout 900 python bench.py --out gpurun_out/bench_phi.json > gpurun_out/bench_phi.log 2>&1; echo "phi rc=$?" >> gpurun_out/bench_phi.log
tail -5 gpurun_out/bench_tiny.log gpurun_out/bench_phi.log
