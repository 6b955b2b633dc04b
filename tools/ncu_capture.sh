#!/bin/bash
# ncu captures used for profiles/ (run on the GPU box from the repo root, one GPU).
#   launches: serialized per-launch durations of ~2 mid-schedule circuits (config 2)
#   full:     one --set full capture each of the decode attention kernel and the gate/up GEMM
# Usage: tools/ncu_capture.sh [launches|full|all]
set -e
OUT=${OUT:-gpurun_out}
mkdir -p "$OUT"
what=${1:-all}
DRV="python tools/step_driver.py --circuits 300"
if [[ $what == launches || $what == all ]]; then
  ncu --metrics gpu__time_duration.sum --clock-control none --launch-skip 70000 --launch-count 600 \
      --csv --log-file "$OUT/launches.csv" $DRV > "$OUT/ncu_launches.log" 2>&1 || true
fi
if [[ $what == full || $what == all ]]; then
  ncu --set full --clock-control none --import-source on -k regex:attn_decode \
      --launch-skip 9000 --launch-count 1 -o "$OUT/attn_decode" -f $DRV > "$OUT/ncu_attn.log" 2>&1 || true
  ncu --set full --clock-control none --import-source on -k regex:gemm_tc_kernel \
      --launch-skip 35842 --launch-count 1 -o "$OUT/gemm_gu" -f $DRV > "$OUT/ncu_gemm.log" 2>&1 || true
fi
