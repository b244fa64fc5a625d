#!/bin/bash
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_xcodec_gpu.py -x -q -m gpu 2>&1 | tail -5
timeout 600 python tools/xc_bench.py > gpurun_out/xc_bench.log 2>&1; grep -E "ratio|decode_GBps|h2d|nc8|nc4" gpurun_out/xc_bench.log
