"""N>1 leg of bench.py: one process per GPU (torchrun), pipeline stage r on GPU r, NCCL hops.

Workload: BASELINE configs[2] as written -- configs/llama8b_4stage_swap.json (Llama-3-8B, 4
stages of 8 layers, 100 ms injected latency per hop, 32 microbatches, KV swap on with the
swap-forcing prompts: 3840-token prompts, 256 generated tokens, prefill_chunk 16384). At N = 2 / 8
the same document with N nodes (same per-node memory, calibration, link and scheduler settings;
the reference planner re-partitions the 32 layers). No field is rewritten and no circuit cap is
applied: the timed run executes every circuit the reference schedule starts before the workload's
bench_duration_s.

Metric = the reference's own (SimReport.output_throughput, sim.cpp:510; windowed_stats,
workload.cpp:82-116): decode tokens at last-stage circuit ends inside [warmup_s, duration) of the
hardware run's real-clock EventTrace (every rank writes its stage's events on the shared host
steady clock; rank 0 merges them, ds_trace_merge) / window length. `steps` = K equal sub-windows
of that window (ms_per_step = window / K); warm-up = W runs of a short schedule prefix (two
circuits per microbatch) from empty KV pools before the measured run. e2e = all decode tokens of
the measured run / host wall time of its ds_session_run call (prefill transient from empty pools
included, sampled ids copied to host every circuit).
"""
import ctypes as C
import json
import os
import sys

CONFIGS = os.path.join(os.path.dirname(os.path.abspath(__file__)), "configs")
METRIC = "generated tokens/sec (whole pipeline) at injected inter-stage latency; roofline fraction"
BASE_CONFIG = "llama8b_4stage_swap.json"


def pipeline_config(n_stages, name=BASE_CONFIG, latency_us=None):
    """The config document with n_stages nodes (identical node/link/scheduler fields)."""
    cfg = json.load(open(os.path.join(CONFIGS, name)))
    node = cfg["nodes"][0]
    cfg["nodes"] = [dict(node, node_id=f"g{i}") for i in range(n_stages)]
    link = cfg["links"][0]
    cfg["links"] = [dict(link, src=f"g{i}", dst=f"g{(i + 1) % n_stages}",
                         latency_us=link["latency_us"] if latency_us is None else latency_us)
                    for i in range(n_stages)]
    return cfg


def arm_config(world):
    """The N>1 arm's `config` (deterministic for a given N; the run-dependent window and counts go
    to `workload_detail`). Read from the config document alone, so bench.py's reference arm emits
    the identical dict without loading the product."""
    nb = json.load(open(os.path.join(CONFIGS, BASE_CONFIG)))["scheduler"]["nb_override"]
    return {"workload": f"Llama-3-8B {world}-stage pipeline on {world}xB200, 100 ms injected "
                        f"latency per hop, {nb} microbatches, KV swap on (configs/{BASE_CONFIG} "
                        f"with {world} nodes, as written)",
            "parallelism": f"pp{world}",
            "hops": "NCCL send/recv over NVLink, one 2-rank communicator per ring link"}


def run_multi(args):
    import torch.distributed as dist

    from bench import ClockSampler, roofline
    from paper_2501_14784_b200 import pipeline as pl
    from paper_2501_14784_b200._native import GpuOpts, check, lib

    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", str(rank)))
    os.environ["NCCL_DEBUG"] = "WARN"  # stdout carries exactly one JSON line (no NCCL version banner)
    if world != args.gpus:
        raise SystemExit(f"--gpus {args.gpus} but WORLD_SIZE {world}: launch with torchrun")
    dist.init_process_group("gloo", init_method="env://", rank=rank, world_size=world)
    ids = [None]
    if rank == 0:
        buf = (C.c_uint8 * (128 * world))()
        for i in range(world):
            one = (C.c_uint8 * 128)()
            check(lib.ds_nccl_unique_id(one))
            C.memmove(C.addressof(buf) + 128 * i, one, 128)
        ids = [bytes(buf)]
    dist.broadcast_object_list(ids, src=0)
    id_buf = (C.c_uint8 * (128 * world)).from_buffer_copy(ids[0])

    cfg = pipeline_config(world)
    txt = json.dumps(cfg)
    plan_txt = pl.plan_config(txt, CONFIGS)
    plan = json.loads(plan_txt)
    nb = plan["n_microbatches"]
    md = pl.model_desc("llama3-8b")
    opts = GpuOpts(device0=local, n_devices=1, real_delay=1, collect_tokens=0, max_circuits=0,
                   weight_seed=pl.WEIGHT_SEED, trace=1)
    h = C.c_void_p()
    check(lib.ds_session_create_rank(txt.encode(), CONFIGS.encode(), b"", -1, -1, C.byref(md),
                                     C.byref(opts), rank, world, id_buf, C.byref(h)))
    out_dir = os.path.join(os.path.dirname(CONFIGS), "gpurun_out", f"bench_n{world}")
    os.makedirs(out_dir, exist_ok=True)

    def run(profile=False, collect=False):
        cap = 1 << 26
        out = C.create_string_buffer(cap)
        check(lib.ds_session_run(h, int(profile), int(collect), out, cap, None))
        return json.loads(out.value.decode())

    t0 = C.c_int64(0)
    try:
        check(lib.ds_session_limit(h, 2 * nb, None))
        for _ in range(args.warmup):
            dist.barrier()
            run()
        check(lib.ds_session_limit(h, 0, None))
        dist.barrier()
        with ClockSampler([local]) as clk:
            r = run(collect=True)
        check(lib.ds_session_limit(h, 0, C.byref(t0)))
        starts = [None] * world
        dist.all_gather_object(starts, t0.value)
        origin = min(starts)
        trace = os.path.join(out_dir, f"rank{rank}.trace")
        need = C.c_size_t(0)
        check(lib.ds_session_trace(h, trace.encode(), origin, 1, 0, 1, None, 0, C.byref(need)))
        dist.barrier()
        check(lib.ds_session_limit(h, 2 * nb, None))
        prof = run(profile=True)
    finally:
        dist.barrier()
        lib.ds_session_destroy(h)
    gathered = [None] * world
    dist.all_gather_object(gathered, {"wall_us": r["wall_us"], "clk": clk.summary(),
                                      "kernels": prof["stages"][0]["kernels"],
                                      "launches": r["launches"], "stage": r["stages"][0],
                                      "d2h": r["d2h_bytes"], "h2d": r["h2d_bytes"],
                                      "swap_wait_us": r["swap_wait_us"],
                                      "tokens": r["decode_tokens"], "circuits": r["circuits"],
                                      "rows": r["rows"]})
    dist.destroy_process_group()
    if rank != 0:
        return None
    merged = os.path.join(out_dir, "hw.trace")
    pl.trace_merge([os.path.join(out_dir, f"rank{i}.trace") for i in range(world)], merged)
    wl = cfg["workload"]
    end_us = 0
    for line in open(merged):
        end_us = max(end_us, int(line.split()[0][2:]))
    w0, w1 = wl["warmup_s"] * 10**6, min(wl["bench_duration_s"] * 10**6, end_us + 1)
    rep = pl.trace_report(merged, world, w0, w1, wl["rng_seed"])
    subs = []
    for k in range(args.steps):  # K equal sub-windows of the measurement window
        a = w0 + (w1 - w0) * k // args.steps
        b = w0 + (w1 - w0) * (k + 1) // args.steps
        subs.append(pl.trace_report(merged, world, a, b, wl["rng_seed"])["output_throughput"])
    open(os.path.join(out_dir, "report.kv"), "w").write(
        pl.report_kv(rep, plan_txt, cfg["links"][0]["latency_us"], "config"))
    import gzip
    import shutil
    with open(merged, "rb") as fi, gzip.open(merged + ".gz", "wb") as fo:
        shutil.copyfileobj(fi, fo)
    for f in [merged] + [os.path.join(out_dir, f"rank{i}.trace") for i in range(world)]:
        os.remove(f)
    try:  # SURVEY.md 8(d) pipeline roofline of this run (tools/pipeline_roofline.py)
        sys.path.insert(0, os.path.join(os.path.dirname(os.path.abspath(__file__)), "tools"))
        from pipeline_roofline import pipeline_roofline
        pr = pipeline_roofline(out_dir, txt)
        pipe_rf = {k: pr[k] for k in ("pipeline_roofline_tokens_per_s", "pipeline_fraction",
                                      "t_roof_stage_us_mean", "decode_rows_per_circuit_mean",
                                      "circuits_in_window")}
    except (Exception, SystemExit) as e:  # reported, never fatal to the bench line
        pipe_rf = {"error": str(e)[:200]}
    sim = pl.sim_config(txt, CONFIGS)
    clocks = gathered[0]["clk"]
    clocks["per_rank_sm_mhz"] = [g["clk"]["sm_mhz"] for g in gathered]
    clocks["reasons"] = sorted({x for g in gathered for x in g["clk"]["reasons"]})
    rf = roofline(gathered[0]["kernels"])
    rf["rank"] = 0
    wall_max = max(g["wall_us"] for g in gathered)
    last = gathered[world - 1]
    return {
        "metric": METRIC, "value": round(rep["output_throughput"], 2),
        "unit": "tokens/s", "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": round((w1 - w0) / 1e3 / args.steps, 3), "higher_is_better": True,
        "scaling": "strong", "vs_baseline": None, "dtype": "bf16",
        "data": "synthetic (random-init weights, counter-RNG prompts; lengths from the reference "
                "generator seed 42)",
        "config": arm_config(world),
        "workload_detail": {"microbatches": nb, "window_us": [w0, w1], "circuits": last["circuits"],
                            "rows": last["rows"]},
        "window": "reference windowed_stats over [warmup_s, min(bench_duration_s, run end)) of the "
                  "real-clock EventTrace (merged over ranks); steps = equal sub-windows",
        "sub_window_tokens_per_s": [round(x, 1) for x in subs],
        "report": {k: rep[k] for k in ("output_tokens", "output_throughput", "mean_bubble_fraction",
                                        "swap_stall_us", "completed_requests")},
        "reference_sim_tokens_per_s": sim["output_throughput"],
        "analytic_bound_tokens_per_s": pl.steady_state_throughput(plan_txt),
        "pipeline_roofline": pipe_rf,
        "e2e": {"value": round(last["tokens"] / (wall_max / 1e6), 2), "unit": "tokens/s",
                "h2d_bytes_per_step": sum(g["h2d"] for g in gathered),
                "d2h_bytes_per_step": last["d2h"],
                "desc": "all decode tokens of the measured run / host wall time of ds_session_run "
                        "(max over ranks; prefill transient included)"},
        "gpu_launches": sum(g["launches"] for g in gathered),
        "roofline": rf, "clocks": clocks,
        "per_rank": [{"device_ms": g["stage"]["device_ms"], "busy_ms": g["stage"]["busy_ms"],
                      "swap_plan_bytes": g["stage"]["swap_plan_bytes"],
                      "swap_in_bytes": g["stage"]["swap_in_bytes"], "topups": g["stage"]["topups"],
                      "swap_wait_us": g["swap_wait_us"]} for g in gathered],
    }
