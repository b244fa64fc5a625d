#!/bin/bash
mkdir -p gpurun_out
timeout 300 python tools/debug_ctl.py > gpurun_out/debug_ctl.txt 2>&1
bash tools/gpu_tests.sh tests
bash tools/ncu_launches.sh
