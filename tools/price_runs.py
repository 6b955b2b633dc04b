#!/usr/bin/env python3
"""Profit block (reference economics) for committed hardware runs.

For each run directory written by tools/run_config.py (summary.json, hw.trace.gz, report.kv):
rebuilds the SimReport from the real-clock hardware trace (ds_trace_report over the report's
window), checks that its report.kv reproduces the committed one byte for byte, then writes
report_priced.kv = report_to_kv with the profit analysis of the given pricing (a config
document's "pricing" object; default: the reference configs' preset, whattomine-8x4090).

  python tools/price_runs.py profiles/r02_70b_8stage_4gpu [more dirs] [--pricing '{"preset": ...}']
"""
import argparse
import gzip
import json
import os
import shutil
import sys
import tempfile

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2501_14784_b200 import pipeline as pl  # noqa: E402

CONFIGS = os.path.join(ROOT, "configs")


def price_run(run_dir, pricing, out_dir=None):
    summary = json.load(open(os.path.join(run_dir, "summary.json")))
    committed = open(os.path.join(run_dir, "report.kv")).read()
    kv = dict(line.split("=", 1) for line in committed.splitlines())
    txt = open(os.path.join(ROOT, summary["config"])).read()
    policy = summary.get("policy") or ""
    lat = int(summary["latency_us"])
    plan = pl.plan_config(txt, CONFIGS, policy=policy or None,
                          latency_us=lat if policy else -1)
    with tempfile.TemporaryDirectory() as td:
        trace = os.path.join(td, "hw.trace")
        with gzip.open(os.path.join(run_dir, "hw.trace.gz"), "rb") as fi, open(trace, "wb") as fo:
            shutil.copyfileobj(fi, fo)
        rep = pl.trace_report(trace, int(kv["n_stages"]), int(kv["window_start_us"]),
                              int(kv["window_end_us"]), int(kv["seed"]))
    name = policy or "config"
    base = pl.report_kv(rep, plan, lat, name)
    if base != committed:
        raise SystemExit(f"{run_dir}: report rebuilt from the hardware trace differs from report.kv")
    priced = pl.report_kv(rep, plan, lat, name, pricing)
    with open(os.path.join(out_dir or run_dir, "report_priced.kv"), "w") as f:
        f.write(priced)
    block = dict(line.split("=", 1) for line in priced[len(base):].splitlines())
    return {"run": run_dir, "pricing": pricing, **block}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("runs", nargs="+")
    ap.add_argument("--pricing", default='{"preset": "whattomine-8x4090"}')
    a = ap.parse_args()
    pricing = json.loads(a.pricing)
    for d in a.runs:
        print(json.dumps(price_run(d, pricing)))


if __name__ == "__main__":
    main()
