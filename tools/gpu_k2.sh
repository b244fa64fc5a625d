#!/bin/bash
mkdir -p gpurun_out
timeout 300 python tools/int4_timeline.py 2>&1 | tail -12
timeout 900 python -m pytest tests/test_kernels_gpu.py -x -q -m gpu -k "int4" 2>&1 | tail -3
