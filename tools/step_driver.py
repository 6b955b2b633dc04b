"""Runs a prefix of the config-2 schedule once (for ncu / compute-sanitizer captures)."""
import argparse
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2501_14784_b200 import pipeline as pl  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--config", default="llama8b_1stage.json")
ap.add_argument("--circuits", type=int, default=400)
ap.add_argument("--runs", type=int, default=1)
a = ap.parse_args()
cfg = os.path.join(ROOT, "configs", a.config)
with pl.Session(open(cfg).read(), os.path.dirname(cfg), n_devices=1, max_circuits=a.circuits) as s:
    for _ in range(a.runs):
        r = s.run()
    print("circuits", r["circuits"], "tokens", r["decode_tokens"], "device_us", r["device_us"])
