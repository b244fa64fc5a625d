#!/bin/bash
# 1-GPU bench + ncu launch list of one Phi generate() (cap 16 = resident, so the list is the compute)
mkdir -p gpurun_out
timeout 900 python bench.py --steps 3 --warmup 3 --out gpurun_out/bench_phi.json > gpurun_out/bench_phi.log 2>&1
tail -c 400 gpurun_out/bench_phi.log; echo
timeout 900 ncu --profile-from-start off --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/launches.csv python tools/profile_run.py --cap 16 --tokens 4 --k 4 > gpurun_out/ncu_launch_run.log 2>&1
python tools/summarize_launches.py gpurun_out/launches.csv > gpurun_out/launches_summary.txt 2>&1; head -25 gpurun_out/launches_summary.txt
