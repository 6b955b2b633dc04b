#!/bin/bash
# Llama-3-70B stage shapes on one B200 (10-layer stage = one of the 8-stage plan): decode circuits
# of 49 rows (the 8-stage plan's microbatch) and 256 rows at context 1024, and one 3840-token
# prompt; then the same command under ncu: per-launch time + DRAM bytes of every attention,
# GEMM and RoPE/KV launch (cold-cache, serialised) -> decode-attention HBM fraction and GEMM
# tensor fraction at 70B shapes.
mkdir -p gpurun_out
CMD="python tools/calibrate_stage.py --model llama3-70b-bf16 --layers 10 --decode 49,256 --prefill 3840 --ctx 1024 --reps 3 --out gpurun_out/cal70_attn.json"
timeout 300 $CMD > gpurun_out/cal70_plain.log 2>&1 &&
timeout 500 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none \
    -k regex:"attn_|gemm_tc|rope_kv" --csv --log-file gpurun_out/cal70_launches.csv $CMD > gpurun_out/cal70_ncu.log 2>&1
echo "rc=$?"; cat gpurun_out/cal70_plain.log; wc -l gpurun_out/cal70_launches.csv
