#!/bin/bash
mkdir -p gpurun_out
timeout 1200 python -m pytest tests/test_kernels_gpu.py tests/test_batch_gpu.py tests/test_engine_gpu.py tests/test_peer_tier_gpu.py tests/test_fullsize_gpu.py -m gpu -x -q 2>&1 | tail -8 > gpurun_out/pytest_iter4.txt
cat gpurun_out/pytest_iter4.txt
timeout 900 python tools/cap_sweep.py --caps 4,16 --k governor --tokens 128 --steps 2 --warmup 1 \
  --out gpurun_out/cap_sweep_iter4.jsonl > gpurun_out/cap_sweep_iter4.log 2>&1
cat gpurun_out/cap_sweep_iter4.jsonl
bash tools/gpu_draft_prof.sh
