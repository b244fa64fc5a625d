#!/bin/bash
# one --set full capture per hot kernel (K3 tcgen05 GEMM, K2 INT4 draft, K1 router, K4 controller, XC decode)
mkdir -p gpurun_out
for k in k_umma_grouped k_umma_int4p k_resid_norm_route k_ctl_verify_layer k_xc_decode; do
  timeout 600 ncu --profile-from-start off --set full --clock-control none --import-source on \
    -k regex:$k -s 2 -c 1 -o gpurun_out/prof_$k python tools/profile_run.py > gpurun_out/ncu_full_$k.log 2>&1
  echo "$k rc=$?" >> gpurun_out/ncu_full_$k.log
done
ls -la gpurun_out/*.ncu-rep
