#!/bin/bash
# round-2 closing evidence (after the draft-step / K3 / GEMV work): headline bench, reference arm,
# peer tier, config 5 (8 streams batched on one GPU), cap sweep, other shapes
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/gpu.txt 2>&1
timeout 1500 python bench.py --out gpurun_out/bench_final2.json > gpurun_out/bench_final2.log 2>&1
tail -c 300 gpurun_out/bench_final2.log; echo
timeout 600 python bench.py --impl reference > gpurun_out/bench_ref_final2.log 2>&1
timeout 900 python bench.py --peer-tier --steps 3 --warmup 3 --no-cpu-baseline --out gpurun_out/bench_peer_final2.json \
  > gpurun_out/bench_peer_final2.log 2>&1
timeout 900 python bench.py --streams 8 --batch --k 3 --steps 2 --warmup 3 --no-cpu-baseline \
  --out gpurun_out/bench_batch8_final2.json > gpurun_out/bench_batch8_final2.log 2>&1
timeout 1500 python tools/cap_sweep.py --caps 4,8,12,14,16 --k governor --tokens 128 --steps 2 --warmup 1 \
  --out gpurun_out/cap_sweep_final2.jsonl > gpurun_out/cap_sweep_final2.log 2>&1
timeout 900 python bench.py --model qwen3 --steps 2 --warmup 3 --tokens 64 --no-cpu-baseline \
  --out gpurun_out/bench_qwen3_final2.json > gpurun_out/bench_qwen3_final2.log 2>&1
timeout 900 python bench.py --model mixtral --steps 2 --warmup 3 --tokens 64 --no-cpu-baseline \
  --out gpurun_out/bench_mixtral_final2.json > gpurun_out/bench_mixtral_final2.log 2>&1
ls gpurun_out
