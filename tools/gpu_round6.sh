#!/bin/bash
mkdir -p gpurun_out
bash tools/gpu_tests.sh tests
timeout 900 python bench.py --steps 3 --warmup 2 --no-cpu-baseline --out gpurun_out/bench_phi.json > gpurun_out/bench_phi.log 2>&1
tail -c 1500 gpurun_out/bench_phi.log
timeout 600 ncu --profile-from-start off --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --cache-control none --csv --log-file gpurun_out/launches_warm.csv python tools/profile_run.py > gpurun_out/ncu_warm.log 2>&1
