#!/usr/bin/env python3
"""Runs one config document end to end on the GPUs of this box, in one process (stage s on GPU
device0 + s % n_devices, peer-copy hops with the injected delay), and writes the reference's
artefacts for it: the real-clock EventTrace, report.kv (report_to_kv, sweep.cpp:146-195), the
reference replay_check verdict on that trace (oracle/_ref) and a summary with per-kernel-kind
roofline numbers from a second, profiled run.

    python tools/run_config.py configs/llama70b_8stage_4gpu.json --gpus 4 --circuits 2000
"""
import argparse
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def load_peaks():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    d = json.load(open(p)) if os.path.exists(p) else {}
    return d.get("hbm_gbs", 6650.0), d.get("bf16_tflops_sustained", 1400.0)


def kernel_kinds(stages):
    """Per kind over all stages: ms, launches, achieved TFLOP/s and GB/s, fractions of peak."""
    hbm, tf = load_peaks()
    agg = {}
    for st in stages:
        for k, v in st["kernels"].items():
            if not isinstance(v, dict) or not v.get("n"):
                continue
            a = agg.setdefault(k, {"ms": 0.0, "n": 0, "flops": 0.0, "bytes": 0.0})
            for f in ("ms", "n", "flops", "bytes"):
                a[f] += v[f]
    out = {}
    for k, a in agg.items():
        s = a["ms"] / 1e3
        if s <= 0:
            continue
        out[k] = {"ms": round(a["ms"], 2), "launch_groups": a["n"],
                  "tflops": round(a["flops"] / s / 1e12, 1), "gbs": round(a["bytes"] / s / 1e9, 1),
                  "tensor_frac": round(a["flops"] / s / 1e12 / tf, 3),
                  "hbm_frac": round(a["bytes"] / s / 1e9 / hbm, 3)}
    return out


def run_one(txt, cdir, policy=None, latency_us=-1, gpus=1, circuits=0, profile=True, out=None):
    """Plan + schedule + execute one config document; returns the summary dict (and writes
    hw.trace / report.kv / summary.json under `out` when given)."""
    import oracle
    from paper_2501_14784_b200 import pipeline as pl
    plan = pl.plan_config(txt, cdir, policy=policy, latency_us=latency_us)
    t0 = time.time()
    sess = pl.Session(txt, cdir, policy=policy, latency_us=latency_us, n_devices=gpus,
                      max_circuits=circuits, trace=True)
    t_build = time.time() - t0
    trace = os.path.join(out or "/tmp", "hw.trace")
    try:
        t0 = time.time()
        gpu = sess.run()
        wall = time.time() - t0
        rep = sess.trace(trace)
        prof = sess.run(profile=True) if profile else None
    finally:
        sess.close()
    lat = latency_us
    if lat < 0:
        links = json.loads(txt).get("links", [])
        lat = links[0]["latency_us"] if links else 0
    # the config's pricing section, when it has one, adds the reference's profit block
    kv = pl.report_kv(rep, plan, lat, policy or "config", json.loads(txt).get("pricing"))
    viol = oracle.Ref().replay_check(trace, plan)
    kinds = {}
    for v in viol:
        kinds[v.split()[0]] = kinds.get(v.split()[0], 0) + 1
    p = json.loads(plan)
    summary = {
        "policy": policy, "latency_us": lat,
        "gpus": gpus, "stages": len(p["stages"]), "n_microbatches": p["n_microbatches"],
        "batch_per_mb": p["stages"][0]["batch_size_per_microbatch"],
        "circuits": gpu["circuits"], "decode_tokens": gpu["decode_tokens"], "rows": gpu["rows"],
        "wall_s": round(wall, 3), "build_s": round(t_build, 1),
        "report": {k: rep[k] for k in ("window_start_us", "window_end_us", "output_tokens",
                                        "output_throughput", "mean_bubble_fraction",
                                        "swap_stall_us", "trace_events", "run_end_us")},
        "analytic_bound_tokens_per_s": pl.steady_state_throughput(plan),
        "reference_sim": {k: v for k, v in pl.sim_config(txt, cdir, policy=policy,
                                                        latency_us=latency_us).items()
                          if k in ("output_throughput", "output_tokens", "swap_stall_us",
                                   "mean_bubble_fraction")},
        "replay_check": {"violations": len(viol), "by_kind": kinds},
        "swap": {"plan_bytes": sum(s["swap_plan_bytes"] for s in gpu["stages"]),
                 "moved_in_bytes": sum(s["swap_in_bytes"] for s in gpu["stages"]),
                 "moved_out_bytes": sum(s["swap_out_bytes"] for s in gpu["stages"]),
                 "topups": sum(s["topups"] for s in gpu["stages"]),
                 "schedule_swap_ins": sum(len(x) for x in gpu["swap_pairs"]),
                 # per schedule swap-in: slot refill vs the plan's bytes (H4: <= plan + 1 page)
                 "refill_over_plan_plus_page": sum(1 for st, pg in zip(gpu["swap_pairs"], gpu["page_bytes"])
                                                   for x in st if x[1] > x[0] + pg),
                 "refill_bytes": sum(x[1] for st in gpu["swap_pairs"] for x in st),
                 "migrated_bytes": sum(x[2] for st in gpu["swap_pairs"] for x in st),
                 "evicted_bytes": sum(x[3] for st in gpu["swap_pairs"] for x in st),
                 "measured_swap_wait_us": gpu["swap_wait_us"]},
        "per_stage": [{"device": s["device"], "computes": s["computes"], "busy_ms": round(s["busy_ms"], 1),
                       "swap_plan_bytes": s["swap_plan_bytes"], "swap_in_bytes": s["swap_in_bytes"],
                       "topups": s["topups"],
                       "not_ready_resident": s["kernels"].get("not_ready_resident"),
                       "not_ready_growth": s["kernels"].get("not_ready_growth")} for s in gpu["stages"]],
    }
    if prof is not None:
        summary["kernels"] = kernel_kinds(prof["stages"])
        summary["kernel_ms_total"] = round(sum(v["ms"] for k, v in summary["kernels"].items()
                                               if k != "swap_wait"), 1)
    if out:
        open(os.path.join(out, "report.kv"), "w").write(kv)
        json.dump(summary, open(os.path.join(out, "summary.json"), "w"), indent=1)
        # keep gpurun_out small (the call returns <= 64 MiB): the trace travels gzipped
        import gzip
        import shutil
        with open(trace, "rb") as fi, gzip.open(trace + ".gz", "wb") as fo:
            shutil.copyfileobj(fi, fo)
        os.remove(trace)
    return summary


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("config")
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--circuits", type=int, default=0, help="executed schedule prefix (0 = all)")
    ap.add_argument("--policy", default=None)
    ap.add_argument("--latency-us", type=int, default=-1)
    ap.add_argument("--no-profile", action="store_true")
    ap.add_argument("--out", default=None)
    a = ap.parse_args()
    cfg_path = os.path.abspath(a.config)
    name = os.path.basename(cfg_path).replace(".json", "")
    if a.policy:
        name += f"_{a.policy}"
    if a.latency_us >= 0:
        name += f"_{a.latency_us // 1000}ms"
    out = a.out or os.path.join(ROOT, "gpurun_out", name)
    os.makedirs(out, exist_ok=True)
    summary = run_one(open(cfg_path).read(), os.path.dirname(cfg_path), a.policy, a.latency_us,
                      a.gpus, a.circuits, not a.no_profile, out)
    summary["config"] = os.path.relpath(cfg_path, ROOT)
    json.dump(summary, open(os.path.join(out, "summary.json"), "w"), indent=1)
    print(json.dumps(summary))


if __name__ == "__main__":
    main()
