#!/bin/bash
mkdir -p gpurun_out
timeout 900 ncu --profile-from-start off --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/launches.csv python tools/profile_run.py "$@" > gpurun_out/ncu_launch_run.log 2>&1
echo "rc=$?" >> gpurun_out/ncu_launch_run.log
tail -3 gpurun_out/ncu_launch_run.log
