#!/bin/bash
# One-GPU pass after the GEMM epilogue changes: GEMM + stage tests, the GEMM phase trace,
# the shape sweep, the N=1 bench and the 8B calibration points.
tag=${1:-r02c}
mkdir -p gpurun_out
python -m pytest tests/test_gpu_gemm.py tests/test_gpu_stage.py tests/test_gpu_pipeline.py -q -x -p no:cacheprovider > gpurun_out/${tag}_tests.log 2>&1
echo "tests rc=$?"; tail -2 gpurun_out/${tag}_tests.log
DS_GEMM_TRACE=1 python tools/gemm_trace.py > gpurun_out/${tag}_gemm_trace.txt 2>&1; grep -E "T N K|epi_main|mma_done" gpurun_out/${tag}_gemm_trace.txt
bash tools/gemm_quick.sh 64,128,180,256,384 > gpurun_out/${tag}_gemm.txt 2>&1; cat gpurun_out/${tag}_gemm.txt
python bench.py --steps 3 --warmup 3 > gpurun_out/${tag}_bench_n1.json 2> gpurun_out/${tag}_bench_n1.err
echo "bench rc=$?"; python -c "import json;d=json.load(open('gpurun_out/${tag}_bench_n1.json'));print(d['value'],d['ms_per_step'],{k:v['ms'] for k,v in d['roofline']['by_kind'].items()})"
python tools/calibrate_stage.py --model llama3-8b --layers 32 --ctx 512 --decode "" \
    --out gpurun_out/${tag}_cal_8b.json > gpurun_out/${tag}_cal_8b.txt 2>&1; echo "cal 8b rc=$?"; cat gpurun_out/${tag}_cal_8b.txt
