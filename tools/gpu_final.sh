#!/bin/bash
# end-of-session evidence: bench line (with the CPU baseline), cap sweep, launch list
mkdir -p gpurun_out
timeout 900 python bench.py --steps 3 --warmup 3 --out gpurun_out/bench_phi.json > gpurun_out/bench_phi.log 2>&1
tail -c 300 gpurun_out/bench_phi.log; echo
timeout 1500 python tools/cap_sweep.py --caps 4,8,12,14,16 --tokens 32 --steps 2 --warmup 1 > gpurun_out/cap_sweep.log 2>&1
tail -5 gpurun_out/cap_sweep.log | cut -c1-200
timeout 900 ncu --profile-from-start off --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/launches.csv python tools/profile_run.py --cap 4 --tokens 4 --k 1 > gpurun_out/ncu_launch_run.log 2>&1
python tools/summarize_launches.py gpurun_out/launches.csv > gpurun_out/launches_summary.txt 2>&1; head -16 gpurun_out/launches_summary.txt
