#!/bin/bash
mkdir -p gpurun_out
timeout 900 python tools/cap_sweep.py --caps 4,16 --k governor --tokens 128 --steps 2 --warmup 1 \
  --out gpurun_out/cap_sweep_iter8.jsonl > gpurun_out/cap_sweep_iter8.log 2>&1
cat gpurun_out/cap_sweep_iter8.jsonl
bash tools/gpu_draft_prof.sh
timeout 1800 python -m pytest tests -m gpu -x -q 2>&1 | tail -6 > gpurun_out/pytest_iter8.txt
cat gpurun_out/pytest_iter8.txt
python __graft_entry__.py smoke > gpurun_out/smoke8.txt 2>&1; echo "smoke rc=$?" >> gpurun_out/smoke8.txt
