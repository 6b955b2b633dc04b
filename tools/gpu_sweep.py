"""Latency x policy sweep of the pipelined path on real GPUs (reference
apply_policy / run_sweep, sweep.cpp:26-43,101-144): for each (hop latency, policy) the reference
planner sizes the pipeline (baseline: no offload, N_B = S; offload: N_B = S with the KV offload
pool; opt: offload with N_B from the latency), the reference scheduler composes the circuits, and
the stage steps run on the GPUs with NCCL hops carrying the injected delay. Reports the
steady-state windowed tok/s (bench_multi.steady_window) next to the reference's own simulated
tok/s (virtual clock, same plan, measured B200 calibration).

    torchrun --nproc-per-node 4 tools/gpu_sweep.py [--latencies 10,50,200] [--rounds 24]
"""
import argparse
import ctypes as C
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch.distributed as dist  # noqa: E402

from bench_multi import CONFIGS, pipeline_config, steady_window  # noqa: E402
from paper_2501_14784_b200 import pipeline as pl  # noqa: E402
from paper_2501_14784_b200._native import GpuOpts, check, lib  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--latencies", default="10,50,200")
ap.add_argument("--policies", default="baseline,offload,opt")
ap.add_argument("--rounds", type=int, default=24, help="circuits per microbatch (opt)")
ap.add_argument("--rounds-few-mb", type=int, default=120,
                help="circuits per microbatch for baseline / offload (N_B = S: each microbatch holds "
                     "~B requests whose prefill must pass before decode dominates)")
ap.add_argument("--out", default=os.path.join(ROOT, "gpurun_out", "gpu_sweep.json"))
a = ap.parse_args()
rank, world = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"])
local = int(os.environ.get("LOCAL_RANK", rank))
dist.init_process_group("gloo")
results = []
for lat_ms in [int(x) for x in a.latencies.split(",")]:
    for policy in a.policies.split(","):
        cfg = pipeline_config(world, latency_us=lat_ms * 1000, nb=0)
        cfg["scheduler"]["nb_override"] = 0
        txt = json.dumps(cfg)
        plan = json.loads(pl.plan_config(txt, CONFIGS, policy=policy))
        nb = plan["n_microbatches"]
        n_circ = nb * (a.rounds if policy == "opt" else a.rounds_few_mb)
        ids = [None]
        if rank == 0:
            buf = b""
            for _ in range(world):
                one = (C.c_uint8 * 128)()
                check(lib.ds_nccl_unique_id(one))
                buf += bytes(one)
            ids = [buf]
        dist.broadcast_object_list(ids, src=0)
        idb = (C.c_uint8 * (128 * world)).from_buffer_copy(ids[0])
        md = pl.model_desc("llama3-8b")
        opts = GpuOpts(device0=local, n_devices=1, real_delay=1, collect_tokens=0,
                       max_circuits=n_circ, weight_seed=pl.WEIGHT_SEED)
        h = C.c_void_p()
        check(lib.ds_session_create_rank(txt.encode(), CONFIGS.encode(), policy.encode(), -1, -1,
                                         C.byref(md), C.byref(opts), rank, world, idb, C.byref(h)))
        out = C.create_string_buffer(1 << 24)
        dist.barrier()
        st = lib.ds_session_run(h, 0, 0, out, 1 << 24, None)
        if st != 0:
            print(f"rank {rank} {policy} {lat_ms} ms failed: {lib.ds_last_error().decode()[:200]}",
                  flush=True)
            os._exit(1)
        r = json.loads(out.value.decode())
        win = None
        if rank == world - 1:
            win = steady_window(txt, n_circ, world, [r["stages"][0]["steps"]])
        got = [None] * world
        dist.all_gather_object(got, win)
        dist.barrier()
        lib.ds_session_destroy(h)
        if rank == 0:
            sim = pl.sim_config(txt, CONFIGS, policy=policy)
            row = {"latency_ms": lat_ms, "policy": policy, "n_microbatches": nb,
                   "batch_per_mb": plan["stages"][0]["batch_size_per_microbatch"],
                   "gpu_tokens_per_s": round(got[world - 1]["tokens_per_s"], 1),
                   "reference_sim_tokens_per_s": round(sim["report"]["output_throughput"], 1)
                   if "report" in sim else sim.get("output_throughput"),
                   "analytic_bound_tokens_per_s": round(pl.steady_state_throughput(json.dumps(plan)), 1),
                   "circuits": n_circ}
            results.append(row)
            print(json.dumps(row), flush=True)
if rank == 0:
    json.dump(results, open(a.out, "w"), indent=1)
dist.destroy_process_group()
