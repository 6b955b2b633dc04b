#!/bin/bash
# Final 4-GPU check: the N=4 bench line exactly as the driver launches it (torchrun, NCCL), stdout
# must be one JSON line.
mkdir -p gpurun_out
timeout 1500 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 \
    --master-port 29613 bench.py --gpus 4 --steps 5 --warmup 3 > gpurun_out/r02f_bench_n4.json 2> gpurun_out/r02f_bench_n4.err
echo "bench n4 rc=$?"; wc -l gpurun_out/r02f_bench_n4.json; tail -c 1500 gpurun_out/r02f_bench_n4.json; tail -3 gpurun_out/r02f_bench_n4.err
