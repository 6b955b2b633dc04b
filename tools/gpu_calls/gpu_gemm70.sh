#!/bin/bash
# 70B stage GEMM shapes in isolation (weights beyond L2, back to back): default plan vs capped
# cluster counts (max_clusters 74 / 64 / 56: whole rounds of 2-CTA tiles, no k-split), with the
# per-CTA phase trace of one launch each.
mkdir -p gpurun_out
DS_GEMM_TRACE=1 timeout 300 python tools/gemm_bench.py 49,256 0,74,64,56 gu70b,down70b,qkv70b,o70b \
  > gpurun_out/gemm70.jsonl 2> gpurun_out/gemm70_trace.txt
echo "rc=$?"
python -c "
import json
for l in open('gpurun_out/gemm70.jsonl'):
  try: d=json.loads(l)
  except Exception: continue
  print(d['shape'], 'mc', d['mc'], 'T', d['T'], d['us'], 'us', d['gbs'], 'GB/s', d['roof_frac'])
"
