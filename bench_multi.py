"""N>1 leg of bench.py: one process per GPU (torchrun), stage r on GPU r, NCCL hops.

Workload: Llama-3-8B cut into N pipeline stages (32/N layers each, reference partition_layers),
100 ms injected latency per hop, 32 microbatches with KV swap enabled (BASELINE configs[2] at
N=4), §5 prompts [0,512] x [0,512], 4096-token prefill chunk. A step replays the first `rounds` circuits of every
microbatch of the reference schedule from empty KV pools. value = generated tokens / max over
ranks of the step's CUDA-event time on the stage stream (idle waits for delayed hops included);
e2e = same on the host clock around the C-ABI call.
"""
import json
import os
import statistics

CONFIGS = os.path.join(os.path.dirname(os.path.abspath(__file__)), "configs")
METRIC = "generated tokens/sec (whole pipeline) at injected inter-stage latency; roofline fraction"


def pipeline_config(n_stages, latency_us=100_000, nb=32):
    cfg = json.load(open(os.path.join(CONFIGS, "llama8b_4stage.json")))
    node = cfg["nodes"][0]
    cfg["nodes"] = [dict(node, node_id=f"g{i}") for i in range(n_stages)]
    link = cfg["links"][0]
    cfg["links"] = [dict(link, src=f"g{i}", dst=f"g{(i + 1) % n_stages}", latency_us=latency_us)
                    for i in range(n_stages)]
    cfg["scheduler"]["nb_override"] = nb
    # a 4096-token prefill chunk per circuit: with the reference default (256) the 32 x B requests
    # admitted at t=0 need ~B circuits of prefill per microbatch before decode dominates
    cfg["scheduler"]["prefill_chunk"] = 4096
    return cfg


def steady_window(cfg_txt, n_circ, world, runs_steps):
    """Reference metric semantics (SimReport.output_throughput, sim.cpp:510; windowed_stats,
    workload.cpp:82-116): decode tokens counted at the last stage's compute ends inside the
    measurement window / window length. The window starts after the first third of the last
    stage's computes (the prefill transient from empty KV pools: warm-up), on the GPU event clock
    of the last stage."""
    from paper_2501_14784_b200 import pipeline as pl
    sched = pl.schedule_config(cfg_txt, CONFIGS, max_circuits=n_circ)
    order = [op[3] for op in sched["ops"][world - 1] if op[0] == 0 and 0 <= op[3] < n_circ]
    n_dec = [c["n_decode"] for c in sched["circuits"]]
    rates = []
    for steps in runs_steps:
        n = min(len(steps), len(order))
        k0 = n // 3
        toks = sum(n_dec[order[k]] for k in range(k0, n))
        ms = steps[n - 1][3] - steps[k0 - 1][3]
        rates.append(toks / (ms / 1e3))
    return {"tokens_per_s": sum(rates) / len(rates),
            "desc": "steady state: decode tokens of the last stage's computes after the first third "
                    "(warm-up from empty KV pools excluded, as the reference's windowed metric) over "
                    "that window on the last stage's GPU event clock; step_tokens_per_s counts the "
                    "whole step"}


def run_multi(args):
    import torch.distributed as dist

    from bench import ClockSampler, roofline
    from paper_2501_14784_b200 import pipeline as pl
    import ctypes as C
    from paper_2501_14784_b200._native import GpuOpts, check, lib

    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", str(rank)))
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
    plan = json.loads(pl.plan_config(txt, CONFIGS))
    nb = plan["n_microbatches"]
    rounds = 30
    md = pl.model_desc("llama3-8b")
    opts = GpuOpts(device0=local, n_devices=1, real_delay=1, collect_tokens=0,
                   max_circuits=nb * rounds, weight_seed=pl.WEIGHT_SEED)
    h = C.c_void_p()
    check(lib.ds_session_create_rank(txt.encode(), CONFIGS.encode(), b"", -1, -1, C.byref(md),
                                     C.byref(opts), rank, world, id_buf, C.byref(h)))

    def run(profile=False):
        cap = 1 << 24
        out = C.create_string_buffer(cap)
        check(lib.ds_session_run(h, int(profile), 0, out, cap, None))
        return json.loads(out.value.decode())

    try:
        for _ in range(args.warmup):
            dist.barrier()
            run()
        runs = []
        with ClockSampler([local]) as clk:
            for _ in range(args.steps):
                dist.barrier()
                runs.append(run())
        dist.barrier()
        prof = run(profile=True)
    finally:
        dist.barrier()
        lib.ds_session_destroy(h)
    dev = [r["device_us"] for r in runs]
    wall = [r["wall_us"] for r in runs]
    window = None
    if rank == world - 1:
        window = steady_window(txt, nb * rounds, world, [r["stages"][0]["steps"] for r in runs])
    gathered = [None] * world
    dist.all_gather_object(gathered, {"dev": dev, "wall": wall, "clk": clk.summary(), "window": window,
                                      "kernels": prof["stages"][0]["kernels"],
                                      "launches": sum(r["launches"] for r in runs),
                                      "stage": prof["stages"][0]})
    dist.destroy_process_group()
    if rank != 0:
        return None
    dev_max = [max(g["dev"][i] for g in gathered) for i in range(args.steps)]
    wall_max = [max(g["wall"][i] for g in gathered) for i in range(args.steps)]
    toks = runs[0]["decode_tokens"]
    clocks = gathered[0]["clk"]
    clocks["per_rank_sm_mhz"] = [g["clk"]["sm_mhz"] for g in gathered]
    clocks["reasons"] = sorted({r for g in gathered for r in g["clk"]["reasons"]})
    rf = roofline(gathered[0]["kernels"])
    rf["rank"] = 0
    win = gathered[world - 1]["window"]
    step_tps = toks * args.steps / (sum(dev_max) / 1e6)
    return {
        "metric": METRIC, "value": round(win["tokens_per_s"], 2),
        "step_tokens_per_s": round(step_tps, 2),
        "window": win["desc"],
        "unit": "tokens/s", "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": round(statistics.mean(dev_max) / 1e3, 3), "higher_is_better": True,
        "scaling": "strong", "vs_baseline": None, "dtype": "bf16",
        "data": "synthetic (random-init weights, counter-RNG prompts; lengths from the reference "
                "generator seed 42)",
        "config": {"workload": f"Llama-3-8B {world}-stage pipeline on {world}xB200, 100 ms injected "
                               f"latency per hop, {nb} microbatches, KV swap enabled, first {rounds} "
                               "circuits of every microbatch",
                   "parallelism": f"pp{world}", "tokens_per_step": toks,
                   "circuits_per_step": runs[0]["circuits"],
                   "analytic_bound_tokens_per_s": pl.steady_state_throughput(json.dumps(plan)),
                   "hops": "NCCL send/recv over NVLink, one 2-rank communicator per ring link"},
        "e2e": {"value": round(toks * args.steps / (sum(wall_max) / 1e6), 2), "unit": "tokens/s",
                "h2d_bytes_per_step": None, "d2h_bytes_per_step": 0},
        "gpu_launches": sum(g["launches"] for g in gathered),
        "roofline": rf, "clocks": clocks,
        "per_rank": [{"device_ms": g["stage"]["device_ms"], "busy_ms": g["stage"]["busy_ms"],
                      "swap_in_bytes": g["stage"]["swap_in_bytes"], "topups": g["stage"]["topups"]}
                     for g in gathered],
    }
