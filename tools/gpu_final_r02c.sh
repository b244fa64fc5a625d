#!/bin/bash
# closing lines on the final code: headline, peer tier, config 5 batched
mkdir -p gpurun_out
timeout 1200 python bench.py --out gpurun_out/bench_final3.json > gpurun_out/bench_final3.log 2>&1
tail -c 300 gpurun_out/bench_final3.log; echo
timeout 900 python bench.py --peer-tier --steps 3 --warmup 3 --no-cpu-baseline --out gpurun_out/bench_peer_final3.json \
  > gpurun_out/bench_peer_final3.log 2>&1
timeout 900 python bench.py --streams 8 --batch --k 3 --steps 2 --warmup 3 --no-cpu-baseline \
  --out gpurun_out/bench_batch8_final3.json > gpurun_out/bench_batch8_final3.log 2>&1
ls gpurun_out | grep final3
