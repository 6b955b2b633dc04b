#!/bin/bash
# GPU suite + smoke + the default N=1 bench (attention timed as prompt / decode groups).
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/f4_gputests.log 2>&1
echo "gpu tests rc=$?"; grep -E 'passed|failed' gpurun_out/f4_gputests.log | tail -2
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/f4_smoke.log 2>&1; echo "smoke rc=$?"; tail -1 gpurun_out/f4_smoke.log
timeout 900 python bench.py > gpurun_out/f4_bench.json 2> gpurun_out/f4_bench.err
echo "bench rc=$?"; python -c "import json;d=json.load(open('gpurun_out/f4_bench.json'));print(d['value'],d['e2e']['value'],d['roofline']['frac'],d['stage_roofline']['frac'],d['gpu_launches'],d['clocks']);print(d['roofline']['by_kind'])"
rm -f gpurun_out/bench_n1.trace
