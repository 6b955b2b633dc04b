#!/bin/bash
# Two-GPU pass: the NCCL ring parity test (verbose) and the N=2 bench line (torchrun).
mkdir -p gpurun_out
python -m pytest tests/test_gpu_multi.py -v -p no:cacheprovider > gpurun_out/r02_nccl_test_n2.log 2>&1
echo "nccl test rc=$?"; grep -E "PASS|FAIL|passed|failed" gpurun_out/r02_nccl_test_n2.log | tail -3
timeout 1500 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 \
    --master-port 29611 bench.py --gpus 2 --steps 5 --warmup 3 > gpurun_out/r02_bench_n2.json 2> gpurun_out/r02_bench_n2.err
echo "bench n2 rc=$?"; tail -c 1500 gpurun_out/r02_bench_n2.json; tail -5 gpurun_out/r02_bench_n2.err
