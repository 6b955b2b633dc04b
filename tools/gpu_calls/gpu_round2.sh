#!/bin/bash
# One-GPU pass after the TMA prompt kernel: GPU tests, the N=1 bench, stage calibration points
# (8B whole model; a 10-layer 70B stage) and the GEMM phase trace.
tag=${1:-r02b}
mkdir -p gpurun_out
python -m pytest tests -m gpu -q -x -p no:cacheprovider > gpurun_out/${tag}_gputests.log 2>&1
echo "gpu tests rc=$?"; tail -3 gpurun_out/${tag}_gputests.log
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/${tag}_smoke.log 2>&1; echo "smoke rc=$?"; tail -2 gpurun_out/${tag}_smoke.log
python bench.py --steps 3 --warmup 3 > gpurun_out/${tag}_bench_n1.json 2> gpurun_out/${tag}_bench_n1.err
echo "bench rc=$?"; python -c "import json;d=json.load(open('gpurun_out/${tag}_bench_n1.json'));print(d['value'],d['ms_per_step'],{k:v['ms'] for k,v in d['roofline']['by_kind'].items()})"
python tools/calibrate_stage.py --model llama3-8b --layers 32 --ctx 512 --decode "" \
    --out gpurun_out/${tag}_cal_8b.json > gpurun_out/${tag}_cal_8b.txt 2>&1; echo "cal 8b rc=$?"; cat gpurun_out/${tag}_cal_8b.txt
python tools/calibrate_stage.py --model llama3-70b-bf16 --first-layer 30 --layers 10 --ctx 512 \
    --out gpurun_out/${tag}_cal_70b10.json > gpurun_out/${tag}_cal_70b10.txt 2>&1; echo "cal 70b rc=$?"; cat gpurun_out/${tag}_cal_70b10.txt
DS_GEMM_TRACE=1 python tools/gemm_trace.py > gpurun_out/${tag}_gemm_trace.txt 2>&1
