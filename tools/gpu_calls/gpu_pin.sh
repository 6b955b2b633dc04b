#!/bin/bash
# Slot policy A/B with the early top-up: DS_SWAP_SLOTS=pin on the two swap configs (4 B200s).
mkdir -p gpurun_out
for c in llama70b_4stage_swap llama8b_4stage_swap; do
  DS_SWAP_SLOTS=pin timeout 1200 python tools/run_config.py configs/$c.json --gpus 4 --no-profile --out gpurun_out/pin_$c > gpurun_out/pin_run_$c.log 2>&1
  echo "$c rc=$?"
  python -c "
import json; d=json.load(open('gpurun_out/pin_$c/summary.json'))
print({k: d[k] for k in ('report','replay_check','wall_s')})
print(d['swap'])"
done
