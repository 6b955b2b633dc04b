"""Runs a config's schedule prefix on one GPU and dumps every stage step's (rows, ms) for
tools/make_calibration.py (measured calibration tables)."""
import argparse
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2501_14784_b200 import pipeline as pl  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--config", required=True)
ap.add_argument("--circuits", type=int, default=0)
ap.add_argument("--runs", type=int, default=2)
ap.add_argument("--out", required=True)
a = ap.parse_args()
cfg = os.path.join(ROOT, "configs", a.config)
runs = []
with pl.Session(open(cfg).read(), os.path.dirname(cfg), n_devices=1, max_circuits=a.circuits) as s:
    s.run()  # warm-up
    for _ in range(a.runs):
        runs.append(s.run())
json.dump({"runs": runs}, open(a.out, "w"))
r = runs[-1]
print("circuits", r["circuits"], "tokens", r["decode_tokens"], "device_us", r["device_us"],
      "steps", sum(len(st["steps"]) for st in r["stages"]))
