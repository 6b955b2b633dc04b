#!/bin/bash
# Validation of the push k-split epilogue (GEMM tests, phase trace, N=1 bench on GPU 0) and the
# swap configs with the pinned lookahead slot choice (4 GPUs).
mkdir -p gpurun_out
CUDA_VISIBLE_DEVICES=0 python -m pytest tests/test_gpu_gemm.py tests/test_gpu_stage.py tests/test_gpu_swap.py -q -x -p no:cacheprovider > gpurun_out/r02e_tests.log 2>&1
echo "tests rc=$?"; tail -2 gpurun_out/r02e_tests.log
CUDA_VISIBLE_DEVICES=0 DS_GEMM_TRACE=1 python tools/gemm_trace.py > gpurun_out/r02e_gemm_trace.txt 2>&1; grep -E "T N K|epi_main|ks_" gpurun_out/r02e_gemm_trace.txt
CUDA_VISIBLE_DEVICES=0 python bench.py --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/r02e_bench_n1.json 2> gpurun_out/r02e_bench_n1.err
echo "bench rc=$?"; python -c "import json;d=json.load(open('gpurun_out/r02e_bench_n1.json'));print(d['value'],d['ms_per_step'],{k:v['ms'] for k,v in d['roofline']['by_kind'].items()})"
for c in llama70b_4stage_swap llama8b_4stage_swap; do
  timeout 900 python tools/run_config.py configs/$c.json --gpus 4 > gpurun_out/run_$c.log 2>&1; echo "$c rc=$?"
  python -c "
import json; d=json.load(open('gpurun_out/$c/summary.json'))
print({k: d[k] for k in ('report','reference_sim','replay_check','swap')})
print([(s['topups'], s['not_ready_resident'], s['not_ready_growth']) for s in d['per_stage']])"
done
