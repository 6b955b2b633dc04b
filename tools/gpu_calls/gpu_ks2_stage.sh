#!/bin/bash
# 70B 10-layer decode step with DS_GEMM_KS2=1 (o / down as 2-way k-split clusters -> RowNorm
# producers, no RMSNorm launches) vs default, then the 70B stage / RowNorm GPU tests under KS2.
mkdir -p gpurun_out
for v in 1 0; do
  DS_GEMM_KS2=$v timeout 40 python tools/calibrate_stage.py --model llama3-70b-bf16 --layers 10 --decode 49,128 --prefill= --ctx 1024 --reps 5 --out gpurun_out/ks2s_$v.json > gpurun_out/ks2s_$v.log 2>&1
  echo "ks2=$v $(tr '\n' ' ' < gpurun_out/ks2s_$v.log)"
done
DS_GEMM_KS2=1 timeout 50 python -m pytest tests/test_gpu_stage.py tests/test_gpu_gemm.py -q -p no:cacheprovider -k "70 or rownorm" > gpurun_out/ks2s_tests.log 2>&1
echo "tests rc=$?"; tail -2 gpurun_out/ks2s_tests.log
