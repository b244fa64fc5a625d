#!/bin/bash
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_kernels_gpu.py -m gpu -x -q -k "int4_tcgen05 or norm_router or combine" 2>&1 | tail -5 | tee gpurun_out/pytest_int4.txt
timeout 600 ncu --profile-from-start off --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --cache-control none --csv --log-file gpurun_out/launches_warm.csv python tools/profile_run.py > gpurun_out/ncu_warm.log 2>&1
python tools/summarize_launches.py gpurun_out/launches_warm.csv
