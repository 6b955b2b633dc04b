#!/usr/bin/env python3
"""SURVEY.md 8(d) pipeline roofline of a committed multi-stage B200 run (tools/run_config.py
output: summary.json + report.kv).

Per circuit of the run's schedule and per stage s (layers L_s of the plan; embedding on the first
stage, LM head on the last): t_roof = max(FLOPs / F, bytes / BW) with FLOPs = 2·T·P_L·L_s +
Σ 4·n_h·d_h·c·L_s (+ 2·R·d·V) and bytes = 2·P_L·L_s + KV read once per row group + KV append +
activations (+ LM head), F / BW the measured sustained tensor / HBM peaks (MEASURED_PEAKS.json).
Circuits = those whose last-stage ComputeEnd falls in the report window [warmup, duration) of the
run's real-clock hardware trace (the k-th last-stage compute of microbatch m is m's k-th schedule
circuit; its (eff_batch, n_decode) are checked against the schedule). T_S := their mean slowest-stage t_roof, B := their
mean decode rows; the pipeline roofline is the reference's steady_state_throughput (sim.cpp:597-604) on them:
nb·B·1e6 / max(nb·T_S, S·T_S + Σ hop latency). Pipeline fraction = the run's windowed
output_throughput / that bound.

  python tools/pipeline_roofline.py profiles/r02_70b_8stage_4gpu [...]
"""
import gzip
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2501_14784_b200 import pipeline as pl  # noqa: E402

CONFIGS = os.path.join(ROOT, "configs")


def peaks():
    try:
        p = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))
        return p["hbm_gbs"], p["bf16_tflops_sustained"], "measured"
    except (OSError, KeyError, ValueError):
        return 6548.5, 1381.7, "round-2 measured values (MEASURED_PEAKS.json absent)"


def pipeline_roofline(run_dir, cfg_txt=None):
    """run_dir: report.kv + hw.trace.gz, and summary.json naming the config unless cfg_txt is
    given (bench.py --gpus N directories: bench_multi.pipeline_config(N))."""
    kv = dict(line.split("=", 1) for line in open(os.path.join(run_dir, "report.kv")).read().splitlines())
    txt = cfg_txt or open(os.path.join(ROOT, json.load(open(os.path.join(run_dir, "summary.json")))["config"])).read()
    plan = json.loads(pl.plan_config(txt, CONFIGS))
    dm = pl.MODEL_DIMS[json.loads(txt)["model"]["name"]]
    d, nh, nkv, dh, ffn, V = (dm["d_model"], dm["n_heads"], dm["n_kv_heads"], dm["d_head"], dm["ffn"],
                              dm["vocab"])
    P_L = d * (nh + 2 * nkv) * dh + nh * dh * d + 3 * d * ffn
    bw, tf, src = peaks()
    stages = [(st["layer_end"] - st["layer_begin"], i == 0, i == len(plan["stages"]) - 1)
              for i, st in enumerate(plan["stages"])]
    with gzip.open(os.path.join(run_dir, "hw.trace.gz"), "rt") as f:
        n_started = sum(1 for line in f if "kind=ComputeStart" in line and " stage=0 " in line)
    sched = pl.schedule_config(txt, CONFIGS, max_circuits=n_started)
    w0, w1 = int(kv["window_start_us"]), int(kv["window_end_us"])
    last_s = str(len(stages) - 1)
    # the k-th last-stage compute of microbatch m is the k-th schedule circuit of m (stages see a
    # microbatch's circuits in order; different microbatches can pass each other between stages)
    by_mb = {}
    for i, c in enumerate(sched["circuits"]):
        by_mb.setdefault(c["mb"], []).append(i)
    seen, open_start, in_window = {}, {}, []
    with gzip.open(os.path.join(run_dir, "hw.trace.gz"), "rt") as f:
        for line in f:
            if "kind=Compute" not in line:
                continue
            e = dict(x.split("=", 1) for x in line.split())
            if e["stage"] != last_s:
                continue
            m = int(e["mb"])
            if e["kind"] == "ComputeStart":
                k = seen.get(m, 0)
                seen[m] = k + 1
                if k >= len(by_mb.get(m, [])):
                    raise SystemExit(f"{run_dir}: the trace does not follow the current plan's "
                                     "schedule (calibration or config changed since the run)")
                i = by_mb[m][k]
                c = sched["circuits"][i]
                if (c["eff_batch"], c["n_decode"]) != (int(e["a"]), int(e["b"])):
                    raise SystemExit(f"{run_dir}: circuit {i} differs between the schedule and the trace")
                open_start[m] = i
            elif w0 <= int(e["t"]) < w1:
                in_window.append(open_start.pop(m))
    t_sum = dec_sum = 0.0
    n = 0
    for i in in_window:
        c = sched["circuits"][i]
        rows = c["rows"]
        T = sum(r[2] for r in rows)
        R = sum(r[3] for r in rows)
        ctx = sum(r[1] * r[2] + r[2] * (r[2] + 1) // 2 for r in rows)
        kv_rows = sum(r[1] + r[2] for r in rows)
        worst = 0.0
        for L, first, last in stages:
            fl = 2.0 * T * P_L * L + 4.0 * nh * dh * ctx * L + (2.0 * R * d * V if last else 0.0)
            by = (2.0 * P_L * L + kv_rows * 4.0 * nkv * dh * L + T * 4.0 * nkv * dh * L + 4.0 * T * d
                  + (2.0 * d * V if last else 0.0) + (2.0 * T * d if first else 0.0))
            worst = max(worst, fl / (tf * 1e12), by / (bw * 1e9))
        t_sum += worst
        dec_sum += c["n_decode"]
        n += 1
    t_s_us = 1e6 * t_sum / n
    b = dec_sum / n
    S, nb = len(stages), plan["n_microbatches"]
    hops = sum(link["latency_us"] for link in plan["ring_links"])
    bound = nb * b * 1e6 / max(nb * t_s_us, S * t_s_us + hops)
    achieved = float(kv["output_throughput"])
    return {"run": os.path.relpath(run_dir, ROOT), "stages": S, "n_microbatches": nb, "window_us": [w0, w1],
            "circuits_in_window": n,
            "t_roof_stage_us_mean": round(t_s_us, 1), "stage_time_us_calibrated": plan["stage_time_us"],
            "decode_rows_per_circuit_mean": round(b, 2), "hop_latency_us_sum": hops,
            "pipeline_roofline_tokens_per_s": round(bound, 2),
            "achieved_output_throughput": achieved, "pipeline_fraction": round(achieved / bound, 4),
            "peaks": {"hbm_gbs": bw, "tflops_sustained": tf, "source": src}}


if __name__ == "__main__":
    for d in sys.argv[1:]:
        cfg = None
        if not os.path.exists(os.path.join(d, "summary.json")):  # a bench.py --gpus N directory
            import bench_multi
            n = int(dict(line.split("=", 1) for line in open(os.path.join(d, "report.kv")))["n_stages"])
            cfg = json.dumps(bench_multi.pipeline_config(n))
        r = pipeline_roofline(d, cfg)
        with open(os.path.join(d, "pipeline_roofline.json"), "w") as f:
            json.dump(r, f, indent=1)
        print(json.dumps(r))
