#!/bin/bash
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_xcodec_gpu.py tests/test_engine_gpu.py -x -q -m gpu 2>&1 | tail -30 > gpurun_out/pytest_xc.txt; cat gpurun_out/pytest_xc.txt
timeout 900 python bench.py --steps 3 --warmup 3 --out gpurun_out/bench_phi_xc.json > gpurun_out/bench_phi_xc.log 2>&1
tail -c 600 gpurun_out/bench_phi_xc.log
