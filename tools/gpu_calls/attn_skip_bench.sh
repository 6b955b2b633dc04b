#!/bin/bash
# Marginal step-time cost of the attention kernels (DS_ATTN_SKIP timing experiments; results invalid).
for m in 0 1 2 4 7; do
  v=$(DS_ATTN_SKIP=$m python bench.py --steps 1 --warmup 3 --no-cpu-baseline 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['ms_per_step'])")
  echo "attn_skip=$m ms_per_step=$v"
done
