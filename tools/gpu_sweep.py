#!/usr/bin/env python3
"""Latency x policy sweep on real GPUs (BASELINE configs[4] shape): the
reference's own matrix (apply_policy / with_uniform_latency / run_sweep, sweep.cpp:26-49,101-144)
with every cell executed on B200s in one process (stage s on GPU s % n; hops carry the injected
delay). Each cell's GPU throughput is the reference metric over the workload window of its
real-clock trace; the reference's virtual-clock prediction of the same cell (same plan, measured
B200 calibration) sits beside it. Writes the reference-format sweep.csv for both, plus per-cell
report.kv files and a JSON summary.

    python tools/gpu_sweep.py configs/llama8b_4stage.json --gpus 4 --latencies 10000,50000,200000 \
        --duration 60 --warmup 20
"""
import argparse
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tools"))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("config")
    ap.add_argument("--gpus", type=int, default=4)
    ap.add_argument("--latencies", default="10000,50000,200000")
    ap.add_argument("--policies", default="baseline,offload,opt")
    ap.add_argument("--duration", type=int, default=0, help="override bench_duration_s (0: as written)")
    ap.add_argument("--warmup", type=int, default=-1, help="override warmup_s (-1: as written)")
    ap.add_argument("--nb", type=int, default=-1, help="override nb_override for opt")
    ap.add_argument("--out", default=os.path.join(ROOT, "gpurun_out", "gpu_sweep"))
    a = ap.parse_args()
    import oracle
    from paper_2501_14784_b200 import pipeline as pl
    from run_config import run_one
    cdir = os.path.dirname(os.path.abspath(a.config))
    cfg = json.load(open(a.config))
    if a.duration:
        cfg["workload"]["bench_duration_s"] = a.duration
    if a.warmup >= 0:
        cfg["workload"]["warmup_s"] = a.warmup
    lats = [int(x) for x in a.latencies.split(",")]
    cfg["sweep"] = {"latencies_us": lats}
    if a.nb >= 0:
        cfg["scheduler"]["nb_override"] = a.nb
    txt = json.dumps(cfg)
    pols = a.policies.split(",")
    os.makedirs(a.out, exist_ok=True)
    cells, gpu_tp, ref_tp = [], [], []
    for p in pols:
        row_g, row_r = [], []
        for lat in lats:
            out = os.path.join(a.out, f"{p}.l{lat}")
            os.makedirs(out, exist_ok=True)
            try:
                s = run_one(txt, cdir, p, lat, a.gpus, 0, False, out)
                os.remove(os.path.join(out, "hw.trace.gz"))  # per-cell traces: report.kv + summary kept
                row_g.append(s["report"]["output_throughput"])
                row_r.append(s["reference_sim"]["output_throughput"])
                cells.append(s)
                print(json.dumps({k: s[k] for k in ("policy", "latency_us", "n_microbatches",
                                                     "batch_per_mb", "circuits", "replay_check")} |
                                 {"gpu_tps": round(row_g[-1], 1), "ref_tps": round(row_r[-1], 1)}),
                      flush=True)
            except Exception as e:  # a failed cell is a "failed" cell, as in the reference
                row_g.append(None)
                row_r.append(None)
                cells.append({"policy": p, "latency_us": lat, "error": str(e)[:300]})
        gpu_tp.append(row_g)
        ref_tp.append(row_r)
    open(os.path.join(a.out, "sweep_gpu.csv"), "w").write(pl.sweep_csv(lats, pols, gpu_tp))
    open(os.path.join(a.out, "sweep_reference.csv"), "w").write(oracle.Ref().sweep_csv(txt, cdir))
    json.dump({"config": os.path.relpath(os.path.abspath(a.config), ROOT),
               "overrides": {"bench_duration_s": cfg["workload"]["bench_duration_s"],
                             "warmup_s": cfg["workload"]["warmup_s"], "latencies_us": lats},
               "cells": cells}, open(os.path.join(a.out, "sweep.json"), "w"), indent=1)


if __name__ == "__main__":
    main()
