#!/bin/bash
# tcgen05 prompt attention iteration: correctness (variant test, stage tests with the kernel
# selected), prefill stage time at 3840 / 16384 rows, one ncu capture on a 3840-token prompt.
mkdir -p gpurun_out
timeout 150 python -m pytest tests/test_gpu_attention_variants.py -q -x -p no:cacheprovider > gpurun_out/tc_variants.log 2>&1
echo "variants rc=$?"; tail -3 gpurun_out/tc_variants.log
DS_ATTN_PROMPT=3 timeout 300 python -m pytest tests/test_gpu_stage.py tests/test_gpu_fulldepth.py -q -x -p no:cacheprovider > gpurun_out/tc_stage.log 2>&1
rc=$?; echo "stage tests (tc) rc=$rc"; tail -3 gpurun_out/tc_stage.log
[ $rc = 0 ] || exit 1
for v in ${VARIANTS:-3 2}; do
  echo "DS_ATTN_PROMPT=$v"; DS_ATTN_PROMPT=$v timeout 300 python tools/calibrate_stage.py --decode "" --prefill 3840,16384 --reps 3 --out gpurun_out/pa_$v.json
done
DS_ATTN_PROMPT=3 timeout 300 ncu --set full --import-source on --clock-control none -k regex:attn_prompt_tc --launch-skip 40 --launch-count 1 -o gpurun_out/pa_tc -f python tools/calibrate_stage.py --decode "" --prefill 3840 --reps 1 > gpurun_out/pa_ncu_tc.log 2>&1
echo "ncu tc rc=$?"; python tools/summarize_ncu.py full gpurun_out/pa_tc.ncu-rep > gpurun_out/pa_ncu_tc.csv 2>&1; cat gpurun_out/pa_ncu_tc.csv
