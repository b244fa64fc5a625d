#!/bin/bash
# round-2 evidence: launch list of a decode with attention at a 256-token context (cap 16, no PCIe)
# and of the cap-4 bench configuration, plus one --set full capture per hot kernel
mkdir -p gpurun_out
P="python tools/profile_run.py --cap 16 --tokens 8 --k 4 --prompt-len 256"
timeout 900 ncu --profile-from-start off --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum \
  --clock-control none --csv --log-file gpurun_out/launches_r02_cap16.csv $P > gpurun_out/launches_r02_cap16.log 2>&1
python tools/summarize_launches.py gpurun_out/launches_r02_cap16.csv > gpurun_out/launches_r02_cap16_summary.txt 2>&1
timeout 900 ncu --profile-from-start off --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum \
  --clock-control none --csv --log-file gpurun_out/launches_r02_cap4.csv python tools/profile_run.py --cap 4 --tokens 4 --k 1 --unique 0 --prompt-len 16 \
  > gpurun_out/launches_r02_cap4.log 2>&1
python tools/summarize_launches.py gpurun_out/launches_r02_cap4.csv > gpurun_out/launches_r02_cap4_summary.txt 2>&1
for spec in "k_attn_partial:40" "k_umma_int4p:40" "k_umma_grouped:60" "k_xc_decode:4" "k_resid_norm_route:40"; do
  k=${spec%%:*}; skip=${spec##*:}
  timeout 600 ncu --profile-from-start off --set full --clock-control none --import-source on \
    -k regex:$k -s $skip -c 1 -o gpurun_out/prof_r02_$k $P > gpurun_out/ncu_full_r02_$k.log 2>&1
  ncu -i gpurun_out/prof_r02_$k.ncu-rep --page details --csv > gpurun_out/ncu_details_r02_$k.csv 2>/dev/null
  ncu -i gpurun_out/prof_r02_$k.ncu-rep --page raw --csv > gpurun_out/ncu_raw_r02_$k.csv 2>/dev/null
done
ls -la gpurun_out/*.ncu-rep
