#!/bin/bash
# round-2 end-of-session evidence: headline bench (+ CPU baselines), reference arm, cap sweep,
# peer tier, the other BASELINE shapes
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/gpu.txt 2>&1
timeout 1500 python bench.py --out gpurun_out/bench_final.json > gpurun_out/bench_final.log 2>&1
timeout 600 python bench.py --impl reference > gpurun_out/bench_ref_final.log 2>&1
timeout 1500 python tools/cap_sweep.py --caps 4,8,12,14,16 --k governor --tokens 128 --steps 2 --warmup 1 \
  --out gpurun_out/cap_sweep_final.jsonl > gpurun_out/cap_sweep_final.log 2>&1
timeout 900 python bench.py --peer-tier --steps 3 --warmup 2 --no-cpu-baseline --out gpurun_out/bench_peer_final.json \
  > gpurun_out/bench_peer_final.log 2>&1
timeout 900 python bench.py --model qwen3 --steps 2 --warmup 1 --tokens 64 --no-cpu-baseline \
  --out gpurun_out/bench_qwen3_final.json > gpurun_out/bench_qwen3_final.log 2>&1
timeout 900 python bench.py --model mixtral --steps 2 --warmup 1 --tokens 64 --no-cpu-baseline \
  --out gpurun_out/bench_mixtral_final.json > gpurun_out/bench_mixtral_final.log 2>&1
