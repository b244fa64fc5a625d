#!/bin/bash
mkdir -p gpurun_out
timeout 1200 python -m pytest tests/test_kernels_gpu.py tests/test_engine_gpu.py tests/test_xcodec_gpu.py -m gpu -x -q 2>&1 | tail -4 > gpurun_out/pytest_iter6.txt
cat gpurun_out/pytest_iter6.txt
timeout 900 python tools/cap_sweep.py --caps 4 --k governor --tokens 128 --steps 2 --warmup 1 \
  --out gpurun_out/cap_sweep_iter6.jsonl > gpurun_out/cap_sweep_iter6.log 2>&1
cat gpurun_out/cap_sweep_iter6.jsonl
bash tools/gpu_final_r02b.sh
