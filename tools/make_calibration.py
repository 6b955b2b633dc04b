"""Measured B200 stage-time table: bench.py --dump writes every stage
step's (rows, ms); this reduces them to the reference's calibration CSV format (batch_size,
total_time_ms with <= 3 decimals; batch strictly increasing, time non-decreasing;
perf_model.cpp:44-83) for the planner and the virtual-clock scheduler."""
import argparse
import json
import statistics

ap = argparse.ArgumentParser()
ap.add_argument("dump")
ap.add_argument("out")
ap.add_argument("--layers", type=int, default=32, help="layers of the measured stage")
ap.add_argument("--model", default="Llama-3-8B")
a = ap.parse_args()
d = json.load(open(a.dump))
steps = []
for r in d["runs"]:
    for st in r["stages"]:
        steps += st["steps"]
buckets = [1, 2, 4, 8, 16, 32, 64, 96, 128, 192, 256, 320, 384, 448, 512]
rows = []
for lo, hi in zip([0] + buckets[:-1], buckets):
    ms = [st[1] for st in steps if lo < st[0] <= hi]
    if len(ms) >= 3:
        rows.append((hi, statistics.median(ms)))
out, last = [], 0.0
for b, ms in rows:
    last = max(last, ms)
    out.append((b, last))
with open(a.out, "w") as f:
    f.write(f"# measured on B200: {a.model} stage of {a.layers} layers, median ms per stage step by "
            f"row bucket (tools/make_calibration.py from bench.py --dump)\n")
    f.write("batch_size,total_time_ms\n")
    for b, ms in out:
        f.write(f"{b},{ms:.3f}\n")
print(open(a.out).read())
