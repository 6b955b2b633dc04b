#!/bin/bash
# A/B of the GEMM L2 weight prefetch (DS_GEMM_L2PF): GEMM shape sweep and the N=1 bench.
mkdir -p gpurun_out
python -m pytest tests/test_gpu_gemm.py -q -x > gpurun_out/ab_gemm_tests.log 2>&1; echo "gemm tests rc=$?"; tail -2 gpurun_out/ab_gemm_tests.log
for pf in 0 48 96; do
  echo "== L2PF=$pf"; DS_GEMM_L2PF=$pf bash tools/gemm_quick.sh 64,128,180,256,384 > gpurun_out/ab_gemm_pf$pf.txt 2>&1; cat gpurun_out/ab_gemm_pf$pf.txt
done
for pf in 0 48; do
  DS_GEMM_L2PF=$pf python bench.py --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/ab_bench_pf$pf.json 2> gpurun_out/ab_bench_pf$pf.err
  python -c "import json;d=json.load(open('gpurun_out/ab_bench_pf$pf.json'));print('bench L2PF=$pf',d['value'],d['ms_per_step'],{k:v['ms'] for k,v in d['roofline']['by_kind'].items()})"
done
