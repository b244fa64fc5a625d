#!/bin/bash
# cap sweep with the XC store + ncu of the persistent K2 and the launch list of one cap-16 generate()
mkdir -p gpurun_out
timeout 1500 python tools/cap_sweep.py --caps 4,8,12,14,16 --tokens 32 --steps 2 --warmup 1 > gpurun_out/cap_sweep.log 2>&1
tail -6 gpurun_out/cap_sweep.log | cut -c1-400
bash tools/gpu_k2prof.sh
timeout 900 ncu --profile-from-start off --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/launches.csv python tools/profile_run.py --cap 16 --tokens 4 --k 4 > gpurun_out/ncu_launch_run.log 2>&1
python tools/summarize_launches.py gpurun_out/launches.csv > gpurun_out/launches_summary.txt 2>&1; head -20 gpurun_out/launches_summary.txt
