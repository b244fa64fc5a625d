#!/bin/bash
# one iteration on the box: kernel + engine parity subset, cap 4/16 sweep, draft launch list,
# batched 8-stream bench (config 5 at N=1)
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_kernels_gpu.py tests/test_batch_gpu.py tests/test_engine_gpu.py -m gpu -x -q 2>&1 | tail -5 > gpurun_out/pytest_iter.txt
cat gpurun_out/pytest_iter.txt
timeout 900 python tools/cap_sweep.py --caps 4,16 --k governor --tokens 128 --steps 2 --warmup 1 \
  --out gpurun_out/cap_sweep_iter.jsonl > gpurun_out/cap_sweep_iter.log 2>&1
cat gpurun_out/cap_sweep_iter.jsonl
bash tools/gpu_draft_prof.sh
timeout 900 python bench.py --streams 8 --batch --k 3 --steps 2 --warmup 1 --tokens 128 --no-cpu-baseline \
  --out gpurun_out/bench_batch8.json > gpurun_out/bench_batch8.log 2>&1
tail -c 600 gpurun_out/bench_batch8.log
