#!/bin/bash
# A/B: L2 prefetch of the down projection's weight stream before griddepcontrol.wait (its CTAs
# start on the SMs the gate/up GEMM's last round leaves idle), N=1 bench alternated.
mkdir -p gpurun_out
for rep in 1 2; do for v in 0 24 64; do
  DS_GEMM_L2PF=$v DS_GEMM_L2PF_KMIN=8192 timeout 400 python bench.py --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/pf_ab_$v$rep.json 2> gpurun_out/pf_ab_$v$rep.err
  python -c "import json;d=json.load(open('gpurun_out/pf_ab_$v$rep.json'));print('pf=$v rep$rep',d['value'],d['clocks']['sm_mhz'],{k:round(v['ms'],1) for k,v in d['roofline']['by_kind'].items()})"
done; done
rm -f gpurun_out/bench_n1.trace
