#!/bin/bash
# Warp-converged MMA issue in the GEMM: GEMM / stage tests, the 8B shape sweep and the N=1 bench.
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_gemm.py tests/test_gpu_stage.py -q -x -p no:cacheprovider > gpurun_out/gw_tests.log 2>&1
rc=$?; echo "tests rc=$rc"; tail -2 gpurun_out/gw_tests.log
[ $rc = 0 ] || exit 1
bash tools/gemm_quick.sh 16,64,128,180,256,1024,4096 > gpurun_out/gw_gemm.txt 2>&1; cat gpurun_out/gw_gemm.txt
timeout 600 python bench.py --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/gw_bench.json 2> gpurun_out/gw_bench.err
echo "bench rc=$?"; python -c "import json;d=json.load(open('gpurun_out/gw_bench.json'));print(d['value'],d['ms_per_step'],d['clocks']['sm_mhz'],{k:v['ms'] for k,v in d['roofline']['by_kind'].items()})"
rm -f gpurun_out/bench_n1.trace
