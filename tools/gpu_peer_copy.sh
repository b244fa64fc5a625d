#!/bin/bash
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_peer_tier_gpu.py tests/test_engine_gpu.py -m gpu -x -q 2>&1 | tail -4 > gpurun_out/pytest_peer.txt
cat gpurun_out/pytest_peer.txt
timeout 900 python bench.py --peer-tier --steps 3 --warmup 3 --no-cpu-baseline --out gpurun_out/bench_peer_final4.json \
  > gpurun_out/bench_peer_final4.log 2>&1
tail -c 400 gpurun_out/bench_peer_final4.log
