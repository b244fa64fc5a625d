#!/bin/bash
# BASELINE configs 2 and 4 (Mixtral, Qwen3 shapes) through bench.py at a 25% per-layer cap
mkdir -p gpurun_out
timeout 1200 python bench.py --model qwen3 --steps 2 --warmup 2 --tokens 16 --no-cpu-baseline --out gpurun_out/bench_qwen3.json > gpurun_out/bench_qwen3.log 2>&1; echo "qwen3 rc=$?"; tail -c 300 gpurun_out/bench_qwen3.log
timeout 1500 python bench.py --model mixtral --steps 2 --warmup 2 --tokens 8 --no-cpu-baseline --out gpurun_out/bench_mixtral.json > gpurun_out/bench_mixtral.log 2>&1; echo "mixtral rc=$?"; tail -c 300 gpurun_out/bench_mixtral.log
