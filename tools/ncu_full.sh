#!/bin/bash
# One `ncu --set full` capture each of the step's kernels (config 2, mid-schedule), summarised
# to CSV (tools/summarize_ncu.py full). GEMM launch index: circuit * 129 + layer * 4 + {0 qkv,
# 1 o, 2 gate-up, 3 down} (32 layers x 4 GEMMs + the LM head per circuit).
OUT=${OUT:-gpurun_out/ncu_r02}
mkdir -p "$OUT"
DRV="python tools/step_driver.py --circuits 320"
C=300; L=10
cap() {  # name regex skip
  ncu --set full --clock-control none --import-source on -k "regex:$2" --launch-skip $3 --launch-count 1 \
      -o "$OUT/$1" -f $DRV > "$OUT/$1.log" 2>&1
  python tools/summarize_ncu.py full "$OUT/$1.ncu-rep" > "$OUT/$1.csv" 2>&1
  echo "== $1"; cat "$OUT/$1.csv"
}
cap gemm_qkv gemm_tc_kernel $((C * 129 + L * 4 + 0))
cap gemm_o gemm_tc_kernel $((C * 129 + L * 4 + 1))
cap gemm_gate_up gemm_tc_kernel $((C * 129 + L * 4 + 2))
cap gemm_down gemm_tc_kernel $((C * 129 + L * 4 + 3))
cap attn_decode attn_decode_tma 9000
cap attn_prompt attn_prompt_tma 3000
cap rmsnorm rmsnorm_kernel 20000
cap rope_kv rope_kv_kernel 10000
