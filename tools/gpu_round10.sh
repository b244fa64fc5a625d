#!/bin/bash
mkdir -p gpurun_out
( timeout 300 python tools/debug_replay.py 31; MSPQ_CTL_NO_STAGING=1 timeout 300 python tools/debug_replay.py 31 ) > gpurun_out/debug_replay.txt 2>&1
tail -40 gpurun_out/debug_replay.txt
timeout 600 python -m pytest tests/test_kernels_gpu.py -x -q -m gpu -k "int4" > gpurun_out/pytest_int4.txt 2>&1; tail -5 gpurun_out/pytest_int4.txt
timeout 300 python tools/int4_timeline.py > gpurun_out/int4_timeline.txt 2>&1; cat gpurun_out/int4_timeline.txt | tail -30
