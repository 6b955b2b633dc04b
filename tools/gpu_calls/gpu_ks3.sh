#!/bin/bash
# A/B of 3-way k-split clusters for the q/k/v projection (DS_GEMM_KS3=1: final bf16 output in the
# GEMM, no k-range planes for the RoPE kernel to sum): GEMM parity tests under KS3, q/k/v shapes,
# then the N=1 bench alternated.
mkdir -p gpurun_out
DS_GEMM_KS3=1 timeout 600 python -m pytest tests/test_gpu_gemm.py tests/test_gpu_stage.py -q -p no:cacheprovider -x > gpurun_out/ks3_tests.log 2>&1
echo "ks3 tests rc=$?"; tail -2 gpurun_out/ks3_tests.log
for v in 0 1; do echo "KS3=$v"; DS_GEMM_KS3=$v bash tools/gemm_quick.sh 16,64,128,180,256 qkv8b; done
for rep in 1 2; do for v in 1 0; do
  DS_GEMM_KS3=$v timeout 400 python bench.py --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/ks3_ab_$v$rep.json 2> gpurun_out/ks3_ab_$v$rep.err
  python -c "import json;d=json.load(open('gpurun_out/ks3_ab_$v$rep.json'));print('ks3=$v rep$rep',d['value'],d['gpu_launches'],d['clocks']['sm_mhz'],{k:round(v['ms'],1) for k,v in d['roofline']['by_kind'].items()})"
done; done
rm -f gpurun_out/bench_n1.trace
