#!/bin/bash
# 70B configs on 4 B200s with the final kernels (tcgen05 prompt attention at G = 8): the 8-stage
# 100 ms config (BASELINE configs[3] workload (i), two stages per GPU) and the 4-stage swap config.
mkdir -p gpurun_out
for c in llama70b_8stage_4gpu llama70b_4stage_swap; do
  timeout 1200 python tools/run_config.py configs/$c.json --gpus 4 --out gpurun_out/f_$c > gpurun_out/f_run_$c.log 2>&1
  echo "$c rc=$?"
  python -c "
import json; d=json.load(open('gpurun_out/f_$c/summary.json'))
print({k: d[k] for k in ('report','reference_sim','replay_check','wall_s')})
print({k: v['ms'] for k, v in d['kernels'].items()})
print(d['swap'])"
done
