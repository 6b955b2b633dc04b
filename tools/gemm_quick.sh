#!/bin/bash
# GEMM microbench summary (shape T us TF/s GB/s roofline-fraction) for the 8B stage shapes.
python tools/gemm_bench.py ${1:-16,64,128,180,256,384,456} 0 ${2:-qkv8b,o8b,gu8b,down8b} 2>&1 | python -c "
import sys,json
for l in sys.stdin:
  try: d=json.loads(l)
  except Exception: print(l.strip()); continue
  print(d['shape'], d['T'], d['us'], d['tflops'], d['gbs'], d['roof_frac'])
"
