#!/bin/bash
# full GPU parity suite + smoke on the final code, control-plane replay bench, cap 4/16 + draft launch list
mkdir -p gpurun_out
timeout 1800 python -m pytest tests -m gpu -x -q 2>&1 | tail -6 > gpurun_out/pytest_iter7.txt
cat gpurun_out/pytest_iter7.txt
python __graft_entry__.py smoke > gpurun_out/smoke7.txt 2>&1; echo "smoke rc=$?" >> gpurun_out/smoke7.txt
timeout 900 python tools/replay_bench.py --out gpurun_out/replay_bench_r02c.jsonl > gpurun_out/replay_bench_r02c.log 2>&1
timeout 900 python tools/cap_sweep.py --caps 4,16 --k governor --tokens 128 --steps 2 --warmup 1 \
  --out gpurun_out/cap_sweep_iter7.jsonl > gpurun_out/cap_sweep_iter7.log 2>&1
cat gpurun_out/cap_sweep_iter7.jsonl
bash tools/gpu_draft_prof.sh
