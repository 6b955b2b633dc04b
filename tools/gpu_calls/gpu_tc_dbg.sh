#!/bin/bash
# timing-only experiments on the tcgen05 prompt kernel (DS_TC_DBG bits skip work; results invalid)
mkdir -p gpurun_out
for d in ${DBGS:-0 1 2 4 6 7}; do
  DS_TC_DBG=$d DS_ATTN_PROMPT=3 timeout 300 ncu --metrics gpu__time_duration.sum,sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active --clock-control none -k regex:attn_prompt_tc --launch-skip 40 --launch-count 4 --csv python tools/calibrate_stage.py --decode "" --prefill 3840 --reps 1 > gpurun_out/tc_dbg_$d.csv 2>/dev/null
  echo "dbg=$d"; grep attn_prompt_tc gpurun_out/tc_dbg_$d.csv | awk -F'","' '{print $(NF-2), $NF}' | head -8
done
