#!/bin/bash
# tcgen05 prompt attention bring-up: variant test, stage/pipeline tests with the kernel selected,
# then the N=1 bench with it (each under its own timeout).
mkdir -p gpurun_out
timeout 150 python -m pytest tests/test_gpu_attention_variants.py -q -x -p no:cacheprovider > gpurun_out/tc_variants.log 2>&1
echo "variants rc=$?"; tail -15 gpurun_out/tc_variants.log
DS_ATTN_PROMPT=3 timeout 300 python -m pytest tests/test_gpu_stage.py tests/test_gpu_pipeline.py tests/test_gpu_fulldepth.py -q -x -p no:cacheprovider > gpurun_out/tc_stage.log 2>&1
echo "stage tests (tc) rc=$?"; tail -15 gpurun_out/tc_stage.log
DS_ATTN_PROMPT=3 timeout 300 python bench.py --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/tc_bench.json 2> gpurun_out/tc_bench.err
echo "bench tc rc=$?"; python -c "import json;d=json.load(open('gpurun_out/tc_bench.json'));print(d['value'],d['ms_per_step'],{k:v['ms'] for k,v in d['roofline']['by_kind'].items()})"
DS_ATTN_PROMPT=3 timeout 300 ncu --set full --clock-control none -k regex:attn_prompt_tc --launch-skip 3000 --launch-count 1 -o gpurun_out/tc_prompt -f python tools/step_driver.py --circuits 320 > gpurun_out/tc_ncu.log 2>&1
python tools/summarize_ncu.py full gpurun_out/tc_prompt.ncu-rep > gpurun_out/tc_prompt_ncu.csv 2>&1; cat gpurun_out/tc_prompt_ncu.csv
timeout 300 python bench.py --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/tc_bench_default.json 2> gpurun_out/tc_bench_default.err
echo "bench default rc=$?"; python -c "import json;d=json.load(open('gpurun_out/tc_bench_default.json'));print(d['value'],d['ms_per_step'],{k:v['ms'] for k,v in d['roofline']['by_kind'].items()})"
