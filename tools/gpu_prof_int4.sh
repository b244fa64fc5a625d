#!/bin/bash
mkdir -p gpurun_out
timeout 600 ncu --profile-from-start off --set full --clock-control none --import-source on -k regex:k_umma_int4 -s 4 -c 1 -o gpurun_out/prof_int4 python tools/profile_run.py > gpurun_out/ncu_int4.log 2>&1
timeout 600 ncu --profile-from-start off --set full --clock-control none --import-source on -k regex:k_ctl_plan_row -s 1 -c 1 -o gpurun_out/prof_plan python tools/profile_run.py > gpurun_out/ncu_plan.log 2>&1
