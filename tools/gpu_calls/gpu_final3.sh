#!/bin/bash
# Round-2 closing one-GPU pass with RowNorm: the default N=1 bench line, the ncu launch list of
# 6000 mid-schedule launches (per-kernel shares), and ncu --set full of a RowNorm consumer GEMM
# (gate/up) and producer GEMM (o) mid-schedule.
mkdir -p gpurun_out/ncu_r02f
timeout 900 python bench.py > gpurun_out/r02f_bench.json 2> gpurun_out/r02f_bench.err
echo "bench rc=$?"; python -c "import json;d=json.load(open('gpurun_out/r02f_bench.json'));print(d['value'],d['e2e']['value'],d['roofline']['frac'],d['stage_roofline']['frac'],d['gpu_launches'],d['clocks'])"
rm -f gpurun_out/bench_n1.trace
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --launch-skip 70000 --launch-count 6000 \
    --csv --log-file gpurun_out/r02f_launches.csv python tools/step_driver.py --circuits 761 > /dev/null 2>&1
echo "launch list rc=$?"; python tools/summarize_ncu.py launches gpurun_out/r02f_launches.csv > gpurun_out/r02f_launch_shares.csv; cat gpurun_out/r02f_launch_shares.csv
OUT=gpurun_out/ncu_r02f
C=300; L=10
for spec in "gemm_o 1" "gemm_gate_up 2"; do
  set -- $spec
  timeout 300 ncu --set full --clock-control none --import-source on -k "regex:gemm_tc_kernel" --launch-skip $((C * 129 + L * 4 + $2)) --launch-count 1 \
      -o "$OUT/$1" -f python tools/step_driver.py --circuits 320 > "$OUT/$1.log" 2>&1
  python tools/summarize_ncu.py full "$OUT/$1.ncu-rep" > "$OUT/$1.csv" 2>&1
  echo "== $1"; cat "$OUT/$1.csv"
done
