#!/bin/bash
# SFU vs FMA-pipe exp2 split in the tcgen05 prompt attention (DS_TC_EXP 0 / 1): correctness and
# prefill stage time at 3840 / 16384 rows, ncu of each.
mkdir -p gpurun_out
for e in 0 1; do
  DS_TC_EXP=$e timeout 150 python -m pytest tests/test_gpu_attention_variants.py -q -x -p no:cacheprovider > gpurun_out/tc_variants_$e.log 2>&1
  echo "exp=$e variants rc=$?"; tail -2 gpurun_out/tc_variants_$e.log
  DS_TC_EXP=$e DS_ATTN_PROMPT=3 timeout 300 python -m pytest tests/test_gpu_stage.py -q -x -p no:cacheprovider > gpurun_out/tc_stage_$e.log 2>&1
  echo "exp=$e stage rc=$?"; tail -2 gpurun_out/tc_stage_$e.log
  DS_TC_EXP=$e DS_ATTN_PROMPT=3 timeout 300 python tools/calibrate_stage.py --decode "" --prefill 3840,16384 --reps 3 --out gpurun_out/pa_e$e.json
  DS_TC_EXP=$e DS_ATTN_PROMPT=3 timeout 300 ncu --set full --import-source on --clock-control none -k regex:attn_prompt_tc --launch-skip 40 --launch-count 1 -o gpurun_out/pa_tc_e$e -f python tools/calibrate_stage.py --decode "" --prefill 3840 --reps 1 > gpurun_out/pa_ncu_e$e.log 2>&1
  python tools/summarize_ncu.py full gpurun_out/pa_tc_e$e.ncu-rep 2>&1 | tail -1
done
