#!/bin/bash
# ncu launch list of one Phi generate() at full residency (cap 16, fixed k) with a 128-token prompt:
# the summary keyed on (kernel, grid) separates the prefill (T = 128) from the draft/verify launches
mkdir -p gpurun_out
K=${K:-4}
timeout 900 ncu --profile-from-start off --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum \
  --clock-control none --csv --log-file gpurun_out/launches_draft.csv \
  python tools/profile_run.py --cap 16 --tokens 10 --k $K --prompt-len 128 > gpurun_out/ncu_draft_run.log 2>&1
echo "rc=$?" >> gpurun_out/ncu_draft_run.log
python tools/summarize_launches.py gpurun_out/launches_draft.csv --grid > gpurun_out/launches_draft_summary.txt 2>&1
head -40 gpurun_out/launches_draft_summary.txt
