#!/bin/bash
# deferred prefetch off/on at Phi caps 8 and 12 (one box)
mkdir -p gpurun_out
for cap in 8 12; do for v in 0 1; do
  MSPQ_PF_DEFER=$v timeout 600 python bench.py --cap $cap --steps 3 --warmup 3 --no-cpu-baseline \
    > gpurun_out/bench_defer_c${cap}_$v.log 2>&1
  tail -1 gpurun_out/bench_defer_c${cap}_$v.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('cap', $cap, 'defer', $v, round(d['value'],3), round(d['path_roofline']['frac'],4))" \
    | tee -a gpurun_out/defer_caps.txt
done; done
