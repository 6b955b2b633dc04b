#!/bin/bash
# Last one-GPU pass after the executor change: whole GPU suite, smoke(), and the default bench
# command exactly as the driver runs it (stdout must be one JSON line).
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/r02g_gputests.log 2>&1
echo "gpu tests rc=$?"; tail -3 gpurun_out/r02g_gputests.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r02g_smoke.log 2>&1; echo "smoke rc=$?"; tail -1 gpurun_out/r02g_smoke.log
timeout 900 python bench.py > gpurun_out/r02g_bench.json 2> gpurun_out/r02g_bench.err
echo "bench rc=$?"; wc -l gpurun_out/r02g_bench.json; python -c "import json;d=json.load(open('gpurun_out/r02g_bench.json'));print(d['value'],d['e2e']['value'],d['roofline']['frac'],d['clocks'])"
rm -f gpurun_out/bench_n1.trace
