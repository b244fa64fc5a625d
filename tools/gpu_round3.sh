#!/bin/bash
mkdir -p gpurun_out
bash tools/gpu_tests.sh tests
bash tools/ncu_launches.sh
