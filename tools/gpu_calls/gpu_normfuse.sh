#!/bin/bash
# RMSNorm split across the residual GEMMs and their consumers (RowNorm): GPU suite (incl. the
# RowNorm GEMM pair tests and the full-depth parity), smoke(), then an N=1 bench A/B on one box (DS_ROWNORM=0 = the separate
# RMSNorm kernel), alternating, twice each.
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/nf_gputests.log 2>&1
echo "gpu tests rc=$?"; grep -E 'passed|failed|Error' gpurun_out/nf_gputests.log | tail -5
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/nf_smoke.log 2>&1; echo "smoke rc=$?"; tail -1 gpurun_out/nf_smoke.log
for rep in 1 2; do for v in 1 0; do
  DS_ROWNORM=$v timeout 400 python bench.py --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/nf_ab_$v$rep.json 2> gpurun_out/nf_ab_$v$rep.err
  python -c "import json;d=json.load(open('gpurun_out/nf_ab_$v$rep.json'));print('rownorm=$v rep$rep',d['value'],d['gpu_launches'],d['clocks']['sm_mhz'],{k:round(v['ms'],1) for k,v in d['roofline']['by_kind'].items()})"
done; done
rm -f gpurun_out/bench_n1.trace
