#!/bin/bash
# Serialized per-kernel launch lists (ncu gpu__time_duration) of three windows of the config-2
# schedule: prefill-heavy start, middle, decode tail. Summaries in $OUT/launches_w*.csv.
OUT=${OUT:-gpurun_out}
mkdir -p "$OUT"
i=0
for skip in 8000 70000 180000; do
  i=$((i+1))
  ncu --metrics gpu__time_duration.sum --clock-control none --launch-skip $skip --launch-count 600 \
      --csv --log-file "$OUT/launches_w$i.csv" python tools/step_driver.py --circuits 761 > /dev/null 2>&1
  python tools/summarize_ncu.py launches "$OUT/launches_w$i.csv" > "$OUT/launch_shares_w$i.csv"
  echo "window $i (launch-skip $skip)"; cat "$OUT/launch_shares_w$i.csv"
done
