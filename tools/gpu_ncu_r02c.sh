#!/bin/bash
# --set full captures of the draft-step kernels on the final code (T = 1, 128-token context)
mkdir -p gpurun_out
P="python tools/profile_run.py --cap 16 --tokens 8 --k 4 --prompt-len 128"
for spec in "k_attn_partial:300" "k_resid_norm_route:600" "k_int4_gemv:40" "k_lm_head:2"; do
  k=${spec%%:*}; skip=${spec##*:}
  timeout 600 ncu --profile-from-start off --set full --clock-control none --import-source on \
    -k regex:$k -s $skip -c 1 -o gpurun_out/prof_r02c_$k $P > gpurun_out/ncu_full_r02c_$k.log 2>&1
  ncu -i gpurun_out/prof_r02c_$k.ncu-rep --page details --csv > gpurun_out/ncu_details_r02c_$k.csv 2>/dev/null
done
ls -la gpurun_out/*.csv | tail
