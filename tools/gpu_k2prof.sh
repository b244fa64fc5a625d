#!/bin/bash
mkdir -p gpurun_out
for sp in "1 4" "2 4" "1 2" "2 8"; do set -- $sp; SP1=$1 SP2=$2 timeout 120 python tools/k2_run.py; done
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/k2_launches.csv python tools/k2_run.py > /dev/null 2>&1
python tools/summarize_launches.py gpurun_out/k2_launches.csv | head -8
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_umma_int4 -s 6 -c 2 -o gpurun_out/prof_k2 python tools/k2_run.py > gpurun_out/prof_k2.log 2>&1
ncu -i gpurun_out/prof_k2.ncu-rep --page details --csv > gpurun_out/prof_k2_details.csv 2>&1
grep -E '"(Duration|DRAM Throughput|Memory Throughput|Achieved Occupancy|Registers Per Thread|Issue Slots Busy|L2 Hit Rate)"' gpurun_out/prof_k2_details.csv | cut -c1-200
