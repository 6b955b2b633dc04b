#!/bin/bash
# 2-way k-split clusters (DS_GEMM_KS2=1: DSMEM reduction in-kernel, so the o / down projections
# become RowNorm producers) vs the default k-range planes, at the 70B o / down decode shapes.
mkdir -p gpurun_out
for v in 0 1; do
  DS_GEMM_KS2=$v timeout 60 python tools/gemm_bench.py 1,49,128,256 0 o70b,down70b > gpurun_out/ks2_$v.jsonl 2>/dev/null
  python -c "
import json
for l in open('gpurun_out/ks2_$v.jsonl'):
  d=json.loads(l); print('ks2=$v', d['shape'], d['T'], d['us'], d['roof_frac'])"
done
