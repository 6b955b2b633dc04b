#!/bin/bash
# Four-GPU pass: N=4 bench line (torchrun, NCCL), the 70B swap config at the shared-link plan,
# the 8B 4-stage swap config (in-process), and the 70B latency x policy sweep (in-process).
mkdir -p gpurun_out
timeout 1200 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 \
    --master-port 29613 bench.py --gpus 4 --steps 5 --warmup 3 > gpurun_out/r02_bench_n4.json 2> gpurun_out/r02_bench_n4.err
echo "bench n4 rc=$?"; tail -c 800 gpurun_out/r02_bench_n4.json; tail -3 gpurun_out/r02_bench_n4.err
for c in llama70b_8stage_swap_4gpu llama8b_4stage_swap; do
  timeout 1200 python tools/run_config.py configs/$c.json --gpus 4 > gpurun_out/run_$c.log 2>&1
  echo "$c rc=$?"; tail -c 300 gpurun_out/run_$c.log
done
timeout 2400 python tools/gpu_sweep.py configs/llama70b_sweep_4gpu.json --gpus 4 --duration 60 --warmup 20 \
    --out gpurun_out/sweep_70b > gpurun_out/r02_sweep_70b.log 2>&1
echo "sweep rc=$?"; tail -12 gpurun_out/r02_sweep_70b.log; cat gpurun_out/sweep_70b/sweep_gpu.csv gpurun_out/sweep_70b/sweep_reference.csv
