#!/bin/bash
# Four-GPU pass (round 2, final calibration tables): N=4 bench line, the 70B 8-stage configs
# (with and without swap), the 8B 4-stage swap config and the 70B latency x policy sweep.
mkdir -p gpurun_out
timeout 1200 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 \
    --master-port 29617 bench.py --gpus 4 --steps 5 --warmup 3 > gpurun_out/r02_bench_n4.json 2> gpurun_out/r02_bench_n4.err
echo "bench n4 rc=$?"; tail -1 gpurun_out/r02_bench_n4.json | head -c 600; echo; tail -3 gpurun_out/r02_bench_n4.err
for c in llama70b_8stage_4gpu llama70b_8stage_swap_4gpu llama8b_4stage_swap; do
  timeout 1200 python tools/run_config.py configs/$c.json --gpus 4 > gpurun_out/run_$c.log 2>&1
  echo "$c rc=$?"; python -c "
import json; d=json.load(open('gpurun_out/$c/summary.json'))
print({k: d[k] for k in ('n_microbatches','batch_per_mb','circuits','report','reference_sim','replay_check','swap')})"
done
timeout 2400 python tools/gpu_sweep.py configs/llama70b_sweep_4gpu.json --gpus 4 --duration 60 --warmup 20 \
    --out gpurun_out/sweep_70b > gpurun_out/r02_sweep_70b.log 2>&1
echo "sweep rc=$?"; tail -12 gpurun_out/r02_sweep_70b.log; cat gpurun_out/sweep_70b/sweep_gpu.csv gpurun_out/sweep_70b/sweep_reference.csv
du -sh gpurun_out
