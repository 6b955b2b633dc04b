#!/bin/bash
# ncu --set full at Llama-3-70B stage shapes (10-layer stage, 49 decode rows at context 1024 --
# the 8-stage plan's microbatch): the gate/up and down GEMMs and the decode attention of layer 5
# in the third step (2 warm-ups first). GEMM launch index = step * 40 + layer * 4 + {0 qkv, 1 o,
# 2 gate/up, 3 down}; attention index = step * 10 + layer.
OUT=gpurun_out/ncu70
mkdir -p $OUT
CMD="python tools/calibrate_stage.py --model llama3-70b-bf16 --layers 10 --decode 49 --prefill= --ctx 1024 --reps 1 --out $OUT/cal.json"
cap() {  # name regex skip
  timeout 300 ncu --set full --clock-control none --import-source on -k "regex:$2" --launch-skip $3 --launch-count 1 \
      -o "$OUT/$1" -f $CMD > "$OUT/$1.log" 2>&1
  python tools/summarize_ncu.py full "$OUT/$1.ncu-rep" > "$OUT/$1.csv" 2>&1
  echo "== $1"; cat "$OUT/$1.csv"
}
timeout 200 $CMD > $OUT/plain.log 2>&1 && {
  cap gemm_gate_up_70b_t49 gemm_tc $((2 * 40 + 5 * 4 + 2))
  cap gemm_down_70b_t49 gemm_tc $((2 * 40 + 5 * 4 + 3))
  cap attn_decode_70b_t49 attn_decode $((2 * 10 + 5))
}
echo "rc=$?"; cat $OUT/plain.log
