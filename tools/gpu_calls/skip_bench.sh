#!/bin/bash
# Marginal step-time cost of each kernel class (DS_SKIP timing experiments; results invalid).
for m in 0 1 2 4 8 11 16 27; do
  v=$(DS_SKIP=$m python bench.py --steps 1 --warmup 3 --no-cpu-baseline 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['ms_per_step'])")
  echo "skip=$m ms_per_step=$v"
done
