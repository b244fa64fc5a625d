#!/bin/bash
# draft GEMV ring A/B + parity subset + cap sweep + launch list + one full capture of the GEMV
mkdir -p gpurun_out
for mdl in phi qwen3 mixtral; do
  for v in 0 2; do
    echo "$mdl variant $v: $(timeout 300 python tools/gemv_bench.py --model $mdl --split2 4 --variant $v 2>&1 | tail -1)" >> gpurun_out/gemv_ring_ab.txt
  done
done
cat gpurun_out/gemv_ring_ab.txt
timeout 1200 python -m pytest tests/test_kernels_gpu.py tests/test_batch_gpu.py tests/test_engine_gpu.py -m gpu -x -q 2>&1 | tail -8 > gpurun_out/pytest_iter5.txt
cat gpurun_out/pytest_iter5.txt
timeout 900 python tools/cap_sweep.py --caps 4,16 --k governor --tokens 128 --steps 2 --warmup 1 \
  --out gpurun_out/cap_sweep_iter5.jsonl > gpurun_out/cap_sweep_iter5.log 2>&1
cat gpurun_out/cap_sweep_iter5.jsonl
bash tools/gpu_draft_prof.sh
P="python tools/profile_run.py --cap 16 --tokens 8 --k 4 --prompt-len 128"
for spec in "k_int4_gemv_ring:40"; do
  k=${spec%%:*}; skip=${spec##*:}
  timeout 600 ncu --profile-from-start off --set full --clock-control none --import-source on \
    -k regex:$k -s $skip -c 1 -o gpurun_out/prof_r02c_$k $P > gpurun_out/ncu_full_r02c_$k.log 2>&1
  ncu -i gpurun_out/prof_r02c_$k.ncu-rep --page details --csv > gpurun_out/ncu_details_r02c_$k.csv 2>/dev/null
  ncu -i gpurun_out/prof_r02c_$k.ncu-rep --page raw --csv > gpurun_out/ncu_raw_r02c_$k.csv 2>/dev/null
done
