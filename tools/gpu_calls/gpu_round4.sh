#!/bin/bash
# One-GPU pass: full GPU tests + smoke, the GEMM phase trace, ncu full captures of every step
# kernel, and the N=1 bench line.
tag=${1:-r02d}
mkdir -p gpurun_out
python -m pytest tests -m gpu -q -x -p no:cacheprovider > gpurun_out/${tag}_gputests.log 2>&1
echo "gpu tests rc=$?"; tail -3 gpurun_out/${tag}_gputests.log
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/${tag}_smoke.log 2>&1; echo "smoke rc=$?"; tail -1 gpurun_out/${tag}_smoke.log
DS_GEMM_TRACE=1 python tools/gemm_trace.py > gpurun_out/${tag}_gemm_trace.txt 2>&1; head -40 gpurun_out/${tag}_gemm_trace.txt
OUT=gpurun_out/ncu_${tag} bash tools/ncu_full.sh > gpurun_out/${tag}_ncu_full.txt 2>&1; echo "ncu rc=$?"; cat gpurun_out/${tag}_ncu_full.txt | cut -c1-400
for f in gpurun_out/ncu_${tag}/*.ncu-rep; do case $f in *gemm_gate_up*|*attn_decode*) ;; *) rm -f $f;; esac; done; du -sh gpurun_out/ncu_${tag}
python bench.py --steps 3 --warmup 3 > gpurun_out/${tag}_bench_n1.json 2> gpurun_out/${tag}_bench_n1.err
echo "bench rc=$?"; python -c "import json;d=json.load(open('gpurun_out/${tag}_bench_n1.json'));print(d['value'],d['ms_per_step'],{k:v['ms'] for k,v in d['roofline']['by_kind'].items()})"
for pol in plan lookahead; do
  DS_SWAP_SLOTS=$pol python tools/run_config.py configs/tiny_2stage_swap.json --gpus 1 --no-profile --out gpurun_out/swap_ab_$pol > gpurun_out/${tag}_swap_$pol.log 2>&1
  python -c "
import json; d=json.load(open('gpurun_out/swap_ab_$pol/summary.json'))
print('$pol', d['report']['output_throughput'], d['report']['swap_stall_us'], {k: d['swap'][k] for k in ('plan_bytes','moved_in_bytes','topups','measured_swap_wait_us','refill_over_plan_plus_page')}, d['replay_check'])"
done
