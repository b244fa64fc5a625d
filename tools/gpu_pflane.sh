#!/bin/bash
# A/B of the opt-in deferred prefetch (MSPQ_PF_DEFER=1) on one box: engine tests with the lane on,
# then alternating 1-GPU bench runs off / on / off / on
mkdir -p gpurun_out
(timeout 900 python -m pytest tests/test_engine_gpu.py -m gpu -x -q 2>&1 | tail -5; timeout 300 python -m pytest tests/test_engine_gpu.py -m gpu -x -q -k prefetch_issue_order 2>&1 | tail -5) | tee gpurun_out/pflane_tests.txt
for v in 0 1 0 1; do
  MSPQ_PF_DEFER=$v timeout 600 python bench.py --steps 4 --warmup 3 --no-cpu-baseline --out gpurun_out/bench_pflane_$v.json \
    > gpurun_out/bench_pflane_$v.log 2>&1
  tail -1 gpurun_out/bench_pflane_$v.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('defer', $v, d['value'], d['e2e']['value'], d['path_roofline']['frac'])" \
    | tee -a gpurun_out/pflane_ab.txt
done
