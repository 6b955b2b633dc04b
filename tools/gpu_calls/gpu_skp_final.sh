#!/bin/bash
# Final defaults (DS_GEMM_SKP=8 at T <= 128): GPU suite + smoke(), then 70B gate/up default vs uncapped.
mkdir -p gpurun_out
timeout 260 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/skpf_gputests.log 2>&1
echo "gpu tests rc=$?"; grep -E 'passed|failed|Error' gpurun_out/skpf_gputests.log | tail -5
timeout 100 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/skpf_smoke.log 2>&1; echo "smoke rc=$?"; tail -1 gpurun_out/skpf_smoke.log
for v in 8 0; do
  DS_GEMM_SKP=$v timeout 60 python tools/gemm_bench.py 1,49,128 0 gu70b,gu8b > gpurun_out/skpf_$v.jsonl 2>/dev/null
  python -c "
import json
for l in open('gpurun_out/skpf_$v.jsonl'):
  d=json.loads(l); print('skp=$v', d['shape'], d['T'], d['us'], d['roof_frac'])"
done
