#!/bin/bash
# Longest-work-first CTA order for attention (DS_ATTN_LPT): N=1 bench A/B on one box (on, off),
# then the GPU suite and smoke() with the default (on).
mkdir -p gpurun_out
for v in 1 0; do
  DS_ATTN_LPT=$v timeout 300 python bench.py --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/lpt_ab_$v.json 2> gpurun_out/lpt_ab_$v.err
  python -c "import json;d=json.load(open('gpurun_out/lpt_ab_$v.json'));print('lpt=$v',d['value'],d['gpu_launches'],d['clocks']['sm_mhz'],{k:round(v['ms'],1) for k,v in d['roofline']['by_kind'].items()})"
done
timeout 400 python -m pytest tests -m gpu -q -x -p no:cacheprovider > gpurun_out/lpt_gputests.log 2>&1
echo "gpu tests rc=$?"; grep -E 'passed|failed|Error' gpurun_out/lpt_gputests.log | tail -5
timeout 200 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/lpt_smoke.log 2>&1; echo "smoke rc=$?"; tail -1 gpurun_out/lpt_smoke.log
rm -f gpurun_out/bench_n1.trace
