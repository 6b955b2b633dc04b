#!/bin/bash
# Prompt attention at the swap-forcing prefill shape (3840-token prompts, chunks of 3840 / 16384
# rows, Llama-3-8B 32 layers): stage time with each prompt kernel, attention share by DS_SKIP,
# and one ncu capture of each kernel on a 3840-token prompt.
mkdir -p gpurun_out
for v in 2 3; do
  echo "DS_ATTN_PROMPT=$v"; DS_ATTN_PROMPT=$v timeout 300 python tools/calibrate_stage.py --decode "" --prefill 3840,16384 --reps 3 --out gpurun_out/pa_$v.json
done
echo "no attention (DS_SKIP=4)"; DS_SKIP=4 timeout 300 python tools/calibrate_stage.py --decode "" --prefill 3840,16384 --reps 3 --out gpurun_out/pa_skip.json
for k in tma tc; do
  v=2; [ $k = tc ] && v=3
  DS_ATTN_PROMPT=$v timeout 300 ncu --set full --clock-control none -k regex:attn_prompt_$k --launch-skip 40 --launch-count 1 -o gpurun_out/pa_$k -f python tools/calibrate_stage.py --decode "" --prefill 3840 --reps 1 --layers 32 > gpurun_out/pa_ncu_$k.log 2>&1
  echo "ncu $k rc=$?"; python tools/summarize_ncu.py full gpurun_out/pa_$k.ncu-rep > gpurun_out/pa_ncu_$k.csv 2>&1; cat gpurun_out/pa_ncu_$k.csv
done
