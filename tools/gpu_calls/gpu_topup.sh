#!/bin/bash
# Early top-up (residency check before the input wait): swap / pipeline / trace GPU tests, then
# the two swap configs on 4 B200s (in-process), without the profiled second run.
mkdir -p gpurun_out
CUDA_VISIBLE_DEVICES=0 timeout 600 python -m pytest tests/test_gpu_swap.py tests/test_gpu_pipeline.py tests/test_gpu_trace.py -q -x -p no:cacheprovider > gpurun_out/topup_tests.log 2>&1
rc=$?; echo "tests rc=$rc"; tail -2 gpurun_out/topup_tests.log
[ $rc = 0 ] || exit 1
for c in llama70b_4stage_swap llama8b_4stage_swap; do
  timeout 1200 python tools/run_config.py configs/$c.json --gpus 4 --no-profile --out gpurun_out/t_$c > gpurun_out/t_run_$c.log 2>&1
  echo "$c rc=$?"
  python -c "
import json; d=json.load(open('gpurun_out/t_$c/summary.json'))
print({k: d[k] for k in ('report','reference_sim','replay_check','wall_s')})
print(d['swap'])"
done
