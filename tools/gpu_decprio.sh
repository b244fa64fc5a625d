#!/bin/bash
# decode-stream priority A/B (MSPQ_DEC_PRIO=lo vs default high), Phi cap 4, one box
mkdir -p gpurun_out
for v in hi lo hi lo; do
  MSPQ_DEC_PRIO=$v timeout 600 python bench.py --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/bench_decprio_$v.log 2>&1
  tail -1 gpurun_out/bench_decprio_$v.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('dec_prio', '$v', round(d['value'],3), round(d['path_roofline']['frac'],4), round(d['roofline']['frac'],3))" \
    | tee -a gpurun_out/decprio_ab.txt
done
