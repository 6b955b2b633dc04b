#!/usr/bin/env python3
"""Benchmark of the B200 stage-step path (BASELINE.json metric: generated tokens/s of the whole
pipeline at injected inter-stage latency, plus a roofline fraction).

N=1 workload (BASELINE configs[1]): Llama-3-8B random-init bf16, one stage on one B200, offline
batch of 256 synthetic prompts (configs/llama8b_1stage.json; lengths from the reference
generator, seed 42). One "step" = the whole offline batch: every circuit the reference scheduler
composes (761 stage steps: chunked prefill + decode) executed on the GPU until all 256 requests
finish. value = generated tokens / device time (CUDA events on the stage stream); e2e = the same
through the C ABI with host buffers (request metadata H2D each step, sampled tokens D2H) on the
host clock.

N>1 (torchrun, one process per GPU): rank 0 drives an N-stage Llama-3-8B pipeline over the N
GPUs with the injected 100 ms hop delay (configs/llama8b_{N}stage_*); the other ranks hold their
GPU for it and exit 0 after the final barrier.

--impl reference: the reference has no GPU or arithmetic for this path; its CPU
implementation of the stage forward is the oracle port (oracle/llama_ref.c) timed on host cores.
"""
import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)
CONFIGS = os.path.join(ROOT, "configs")
METRIC = "generated tokens/sec (whole pipeline) at injected inter-stage latency; roofline fraction"

SMI_FIELDS = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
              "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")


class ClockSampler:
    """nvidia-smi clocks + throttle reasons during the timed region (B200_PROFILING.md)."""

    def __init__(self, gpus):
        self.gpus = gpus
        self.rows = []
        self.proc = None

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", f"--id={','.join(str(g) for g in self.gpus)}",
                 f"--query-gpu={SMI_FIELDS}", "--format=csv,noheader,nounits", "-lms", "200"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            threading.Thread(target=self._read, daemon=True).start()
        except OSError:
            self.proc = None
        return self

    def _read(self):
        for line in self.proc.stdout:
            self.rows.append([x.strip() for x in line.split(",")])

    def __exit__(self, *a):
        if self.proc:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except subprocess.TimeoutExpired:
                self.proc.kill()

    def summary(self):
        if not self.rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        sm, mx, reasons = [], [], set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for r in self.rows:
            try:
                sm.append(float(r[0]))
                mx.append(float(r[1]))
            except (ValueError, IndexError):
                continue
            for k, n in enumerate(names):
                if len(r) > 4 + k and r[4 + k].lower().startswith("active"):
                    reasons.add(n)
        loaded = [s for s in sm if s > 0.5 * max(sm)] if sm else []
        return {"sm_mhz": statistics.median(loaded) if loaded else None,
                "sm_max_mhz": max(mx) if mx else None, "reasons": sorted(reasons),
                "samples": len(sm)}


def load_peaks():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(p):
        d = json.load(open(p))
        return d["hbm_gbs"], d["bf16_tflops"], d.get("bf16_tflops_sustained", d["bf16_tflops"]), "measured"
    return 6650.0, 1590.0, 1400.0, "fallback"


NCU_FULL = {"gemm_gate_up": "r02_ncu_full_gemm_gate_up.csv", "attention_decode": "r02_ncu_full_attn_decode.csv",
            "attention_prompt": "r02_ncu_full_attn_prompt_tc.csv",
            "gemm_down": "r02_ncu_full_gemm_down.csv", "gemm_o": "r02_ncu_full_gemm_o.csv",
            "gemm_qkv": "r02_ncu_full_gemm_qkv.csv"}


def ncu_traffic(kind):
    """dram__bytes_read + dram__bytes_write of one launch of this kernel kind from the committed
    `ncu --set full` capture under profiles/ (a mid-schedule launch; compare with
    algorithmic_bytes_per_launch, which averages every launch of the step)."""
    name = NCU_FULL.get(kind)
    path = os.path.join(ROOT, "profiles", name) if name else None
    if not path or not os.path.exists(path):
        return None, None
    import csv
    rows = list(csv.reader(open(path)))
    hdr, unit, val = rows[0], rows[1], rows[2]
    scale = {"byte": 1.0, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}
    tot = 0.0
    for key in ("dram__bytes_read.sum", "dram__bytes_write.sum"):
        i = hdr.index(key)
        tot += float(val[i].replace(",", "")) * scale.get(unit[i], 1.0)
    return tot, f"bytes per launch, profiles/{name} (one mid-schedule launch of {val[0]})"


def roofline(kernels):
    """Dominant launch group of the profiled run: algorithmic work / its summed CUDA-event time."""
    hbm, tf_burst, tf_sus, src = load_peaks()
    kinds = {k: v for k, v in kernels.items()
             if isinstance(v, dict) and v.get("n") and k != "swap_wait"}  # swap_wait: not a kernel
    dom = max(kinds, key=lambda k: kinds[k]["ms"])
    v = kinds[dom]
    sec = v["ms"] / 1e3
    intensity = v["flops"] / max(v["bytes"], 1.0)
    ridge = tf_sus * 1e12 / (hbm * 1e9)
    if intensity > ridge:
        ach, peak, unit, bound = v["flops"] / sec / 1e12, tf_sus, "TFLOP/s", "tensor"
    else:
        ach, peak, unit, bound = v["bytes"] / sec / 1e9, hbm, "GB/s", "hbm"
    total_ms = sum(x["ms"] for x in kinds.values())
    traffic, traffic_note = ncu_traffic(dom)
    return {"kernel": dom, "bound": bound, "achieved": round(ach, 2), "peak": peak, "unit": unit,
            "frac": round(ach / peak, 4), "traffic": traffic, "traffic_note": traffic_note,
            "peak_source": src,
            "share_of_step": round(v["ms"] / total_ms, 4), "launches": v["n"],
            "algorithmic_flops_per_launch": v["flops"] / v["n"],
            "algorithmic_bytes_per_launch": v["bytes"] / v["n"],
            "avg_launch_ms": v["ms"] / v["n"],
            "by_kind": {k: {"ms": round(x["ms"], 3), "n": x["n"],
                            "tflops": round(x["flops"] / (x["ms"] / 1e3) / 1e12, 2),
                            "gbs": round(x["bytes"] / (x["ms"] / 1e3) / 1e9, 1)}
                        for k, x in kinds.items()}}


def stage_roofline(cfg_txt, model="llama3-8b"):
    """SURVEY.md 8(d) stage roofline of the schedule the run executes: per circuit
    t_roof = max(FLOPs / F_sustained, bytes / BW) with FLOPs = 2·T·P_L·L + Σ_positions 4·n_h·d_h·c·L
    + 2·R·d·V and bytes = weights + KV read once per request row group (c = group end) + KV
    append + LM head + activations; returns the per-step sum."""
    from paper_2501_14784_b200 import pipeline as pl
    hbm, _, tf_sus, _ = load_peaks()
    dm = pl.MODEL_DIMS[model]
    d, L, nh, nkv, dh, ffn, V = (dm["d_model"], dm["n_layers"], dm["n_heads"], dm["n_kv_heads"],
                                 dm["d_head"], dm["ffn"], dm["vocab"])
    P_L = d * (nh + 2 * nkv) * dh + nh * dh * d + 3 * d * ffn
    sched = pl.schedule_config(cfg_txt, CONFIGS)
    t = fl_all = by_all = 0.0
    for c in sched["circuits"]:
        rows = c["rows"]
        T = sum(r[2] for r in rows)
        R = sum(r[3] for r in rows)
        ctx = sum(r[1] * r[2] + r[2] * (r[2] + 1) // 2 for r in rows)
        fl = 2.0 * T * P_L * L + 4.0 * nh * dh * ctx * L + 2.0 * R * d * V
        by = (2.0 * P_L * L + sum(r[1] + r[2] for r in rows) * 4.0 * nkv * dh * L
              + T * 4.0 * nkv * dh * L + 2.0 * d * V + 4.0 * T * d)
        t += max(fl / (tf_sus * 1e12), by / (hbm * 1e9))
        fl_all += fl
        by_all += by
    return {"t_roof_s_per_step": round(t, 4), "flops_per_step": fl_all, "bytes_per_step": by_all,
            "peaks": {"tflops_sustained": tf_sus, "hbm_gbs": hbm}}


SCHEDULE_FIXTURE = os.path.join(CONFIGS, "llama8b_1stage.schedule.json.gz")
WORKLOAD = ("Llama-3-8B 1 stage on 1xB200, offline batch of 256 prompts "
            "(BASELINE configs[1], configs/llama8b_1stage.json)")
ARM_CONFIG = {"workload": WORKLOAD, "model": "Llama-3-8B (random-init bf16)", "prompts": 256,
              "parallelism": "pp1"}


def systematic_sample(n_total, k):
    """k circuit indices spread evenly over the schedule (systematic sample: every phase of the
    offline batch -- prefill-heavy start, mixed middle, decode tail -- in proportion)."""
    return sorted({min(n_total - 1, int((j + 0.5) * n_total / k)) for j in range(k)})


def time_pipesim(cfg_path):
    """The reference CPU path itself: pipesim run() (oracle/_ref) on the same config, one core."""
    r = subprocess.run(["taskset", "-c", "0", sys.executable,
                        os.path.join(ROOT, "oracle", "time_pipesim.py"), cfg_path],
                       capture_output=True, text=True, timeout=600)
    if r.returncode != 0:
        return {"error": (r.stderr or r.stdout)[-300:]}
    return json.loads(r.stdout.strip().splitlines()[-1])


def oracle_circuits(indices, warmup=0):
    """CPU stage forward (oracle/llama_ref.c, OpenMP on all host cores) on the schedule's own
    circuits: all 32 layers + embedding + LM head, exact rows. Returns per-circuit seconds and
    decode rows. No product code is loaded (the schedule comes from the committed fixture)."""
    import oracle
    circs = oracle.load_schedule_fixture(SCHEDULE_FIXTURE)
    slots = 1 + max(r[0] for c in circs for r in c["rows"])
    tm = oracle.CircuitTimer(oracle.MODEL_DIMS["llama3-8b"], oracle.WEIGHT_SEED, slots)
    try:
        small = min(range(len(circs)), key=lambda i: circs[i]["eff_batch"])
        for _ in range(warmup):
            tm.time(circs[small])
        out = [(i, tm.time(circs[i]), circs[i]["n_decode"], circs[i]["eff_batch"]) for i in indices]
    finally:
        tm.close()
    return out, len(circs), sum(c["n_decode"] for c in circs)


def cpu_baseline(k=2):
    """Bounded CPU baseline for our arm's line (~10-30 s on the GPU box's host): the oracle on k
    systematically sampled circuits of the same schedule (no layer extrapolation), plus
    pipesim run() on one core."""
    idx = systematic_sample(761, k)
    res, circs_n, toks = oracle_circuits(idx)
    t = sum(x[1] for x in res)
    dec = sum(x[2] for x in res)
    return {"value": round(dec / t, 3) if dec else None, "unit": "tokens/s", "cores": os.cpu_count(),
            "kind": "port",
            "sample": f"oracle/llama_ref.c, all 32 layers + LM head, on circuits {idx} of the "
                      f"{circs_n}-circuit schedule (their exact rows): {dec} decode rows in "
                      f"{t:.2f} s; tok/s = decode rows / CPU seconds",
            "est_step_s": round(t * circs_n / len(idx), 1),
            "pipesim": time_pipesim(os.path.join(CONFIGS, "llama8b_1stage.json"))}


def run_single(args):
    from paper_2501_14784_b200 import pipeline as pl
    cfg_path = os.path.join(CONFIGS, "llama8b_1stage.json")
    txt = open(cfg_path).read()
    sess = pl.Session(txt, CONFIGS, n_devices=1, real_delay=True, trace=True)
    try:
        for _ in range(args.warmup):
            sess.run()
        runs = []
        with ClockSampler([0]) as clk:
            for _ in range(args.steps):
                runs.append(sess.run(collect_tokens=True))
        # the last timed run as the reference's SimResult: real-clock trace + SimReport
        os.makedirs(os.path.join(ROOT, "gpurun_out"), exist_ok=True)
        hw_report = sess.trace(os.path.join(ROOT, "gpurun_out", "bench_n1.trace"))
        prof = sess.run(profile=True)
    finally:
        sess.close()
    toks = sum(r["decode_tokens"] for r in runs)
    dev_s = sum(r["device_us"] for r in runs) / 1e6
    wall_s = sum(r["wall_us"] for r in runs) / 1e6
    h2d = sum(r["h2d_bytes"] for r in runs)  # per run (the stage counter resets every run)
    rf = roofline(prof["stages"][0]["kernels"])
    out = {
        "metric": METRIC, "value": round(toks / dev_s, 2), "unit": "tokens/s", "n_gpus": 1,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": round(dev_s * 1e3 / args.steps, 3),
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "bf16",
        "data": "synthetic (random-init weights, counter-RNG prompts; lengths from the reference "
                "generator seed 42)",
        "config": dict(ARM_CONFIG),
        "workload_detail": {"circuits_per_step": runs[0]["circuits"],
                            "tokens_per_step": runs[0]["decode_tokens"],
                            "rows_per_step": runs[0]["rows"],
                            "l2": "inputs larger than L2 (16 GB of weights streamed per circuit)"},
        "e2e": {"value": round(toks / wall_s, 2), "unit": "tokens/s",
                "h2d_bytes_per_step": int(h2d / max(len(runs), 1)) if h2d else None,
                "d2h_bytes_per_step": runs[0]["d2h_bytes"]},
        "gpu_launches": sum(r["launches"] for r in runs),
        "report": {"desc": "SimReport of the last timed run from its real-clock EventTrace "
                           "(ds_session_trace; window = [0, run end): the offline batch's makespan)",
                   **{k: hw_report[k] for k in ("output_tokens", "output_throughput", "window_end_us",
                                                 "mean_bubble_fraction", "completed_requests",
                                                 "trace_events")}},
        "roofline": rf,
        "clocks": clk.summary(),
    }
    try:
        sr = stage_roofline(txt)
        sr["frac"] = round(sr["t_roof_s_per_step"] / (dev_s / args.steps), 4)
        out["stage_roofline"] = sr
    except Exception as e:
        out["stage_roofline"] = {"error": str(e)[:200]}
    if not args.no_cpu_baseline:
        try:
            out["cpu_baseline"] = cpu_baseline()
        except Exception as e:  # the baseline is reported, never the product
            out["cpu_baseline"] = {"value": None, "error": str(e)[:200]}
    if args.dump:
        json.dump({"runs": runs, "profile": prof}, open(args.dump, "w"))
    return out


def run_reference(args):
    """The reference's CPU implementation of the path on the box's host cores, same workload,
    metric and config as our arm. The stage forward has no arithmetic in the reference
    (SURVEY.md 0), so its CPU implementation is the oracle port (oracle/llama_ref.c, every core):
    each step times one circuit of the real schedule at full depth (systematic sample over the
    761 circuits, K steps = K evenly spaced circuits); value = decode rows / CPU seconds over the
    timed circuits. The reference's own engine, pipesim run(), is timed beside it on one core.
    Nothing from the product package is imported or loaded."""
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return None
    world = int(os.environ.get("WORLD_SIZE", "1"))
    n = max(world, args.gpus)
    config = dict(ARM_CONFIG)
    if n > 1:  # our arm's N>1 config (same dict); the CPU has no stage split: whole-model rows
        from bench_multi import arm_config
        config = arm_config(n)
    idx = systematic_sample(761, args.steps)
    res, n_circ, toks = oracle_circuits(idx, warmup=args.warmup)
    t = sum(x[1] for x in res)
    dec = sum(x[2] for x in res)
    v = round(dec / t, 3)
    return {"impl": "reference", "metric": METRIC, "value": v, "unit": "tokens/s",
            "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup,
            "ms_per_step": round(1e3 * t / len(res), 3),
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "bf16",
            "data": "synthetic (random-init weights, counter-RNG prompts; lengths from the reference "
                    "generator seed 42)",
            "config": config,
            "cpu_baseline": {"value": v, "unit": "tokens/s", "cores": os.cpu_count(), "kind": "port",
                             "sample": f"oracle/llama_ref.c (OpenMP, {os.cpu_count()} threads), all 32 "
                                       f"layers + embedding + LM head, one circuit per step: "
                                       f"circuits {idx} of {n_circ} (exact rows; warm-up "
                                       f"{args.warmup} x the smallest circuit); {dec} decode rows "
                                       f"in {t:.2f} s" + (
                                           "; at N > 1 the same full-depth circuits of the 8B "
                                           "offline schedule: one host's cores run the whole "
                                           "model whatever the stage split" if n > 1 else ""),
                             "per_circuit": [{"circuit": i, "s": round(x, 3), "decode_rows": d,
                                              "rows": e} for i, x, d, e in res],
                             "est_whole_batch_s": round(t * n_circ / len(res), 1)},
            "pipesim": time_pipesim(os.path.join(CONFIGS, "llama8b_1stage.json")),
            "e2e": {"value": v, "unit": "tokens/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}


# timing-experiment switches that skip work (their results are invalid): the bench refuses them
INVALIDATING_ENV = ("DS_SKIP", "DS_ATTN_SKIP", "DS_GEMM_NOFINISH", "DS_GEMM_TRACE", "DS_TC_DBG")


def ds_env():
    """Every DS_* override in effect (recorded in the JSON line)."""
    return {k: v for k, v in sorted(os.environ.items()) if k.startswith("DS_")}


class StdoutToStderr:
    """fd-level redirect of stdout to stderr while the run executes, so that anything native code
    prints (NCCL's version banner, CUDA library notices) cannot join the one JSON line on stdout."""

    def __enter__(self):
        sys.stdout.flush()
        self.saved = os.dup(1)
        os.dup2(2, 1)
        return self

    def __exit__(self, *exc):
        sys.stdout.flush()
        os.dup2(self.saved, 1)
        os.close(self.saved)
        return False


def main():
    bad = [k for k in INVALIDATING_ENV if os.environ.get(k) not in (None, "", "0")]
    if bad:
        sys.exit(f"bench.py: {', '.join(bad)} set -- these skip kernels or their finish step and "
                 "invalidate every number; unset them")
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=3)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--dump", default=None, help="write per-run reports (steps, kernels) here")
    args = ap.parse_args()
    if args.impl == "reference":
        with StdoutToStderr():
            out = run_reference(args)
        if out is not None:
            print(json.dumps(out))
        return
    world = int(os.environ.get("WORLD_SIZE", "1"))
    with StdoutToStderr():
        if world > 1 or args.gpus > 1:
            from bench_multi import run_multi
            out = run_multi(args)
        else:
            out = run_single(args)
    if out is not None:
        out["ds_env"] = ds_env()
        print(json.dumps(out))


if __name__ == "__main__":
    main()
