#!/bin/bash
# decode grid per chunk A/B (MSPQ_DEC_CTAS), Phi cap 4, one box
mkdir -p gpurun_out
for v in 256 128 256 128; do
  MSPQ_DEC_CTAS=$v timeout 600 python bench.py --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/bench_decctas_$v.log 2>&1
  tail -1 gpurun_out/bench_decctas_$v.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('dec_ctas', $v, round(d['value'],3), round(d['path_roofline']['frac'],4), round(d['roofline']['frac'],3))" \
    | tee -a gpurun_out/decctas_ab.txt
done
