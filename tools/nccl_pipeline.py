"""Small one-process-per-GPU pipeline run (torchrun) for debugging the NCCL hop path."""
import ctypes as C
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch.distributed as dist  # noqa: E402

from paper_2501_14784_b200 import pipeline as pl  # noqa: E402
from paper_2501_14784_b200._native import GpuOpts, check, lib  # noqa: E402

cfg_name = sys.argv[1] if len(sys.argv) > 1 else "tiny_2stage.json"
n_circ = int(sys.argv[2]) if len(sys.argv) > 2 else 40
profile = int(sys.argv[3]) if len(sys.argv) > 3 else 0  # 1: CUDA events per launch group + swap waits
rank, world = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"])
dist.init_process_group("gloo")
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
cdir = os.path.join(ROOT, "configs")
cfg = json.load(open(os.path.join(cdir, cfg_name)))
if len(cfg["nodes"]) != world:
    node, link = cfg["nodes"][0], cfg["links"][0]
    cfg["nodes"] = [dict(node, node_id=f"g{i}") for i in range(world)]
    cfg["links"] = [dict(link, src=f"g{i}", dst=f"g{(i + 1) % world}") for i in range(world)]
txt = json.dumps(cfg)
md = pl.model_desc(cfg["model"]["name"])
opts = GpuOpts(device0=int(os.environ.get("LOCAL_RANK", rank)), n_devices=1, real_delay=1,
               collect_tokens=1, max_circuits=n_circ, weight_seed=pl.WEIGHT_SEED)
h = C.c_void_p()
check(lib.ds_session_create_rank(txt.encode(), cdir.encode(), b"", -1, -1, C.byref(md), C.byref(opts),
                                 rank, world, idb, C.byref(h)))
print(f"rank {rank} session ready", flush=True)
out = C.create_string_buffer(1 << 24)
st = lib.ds_session_run(h, profile, 1, out, 1 << 24, None)
r = json.loads(out.value.decode() or "{}")
print(f"rank {rank} status {st} err={lib.ds_last_error().decode()[:200]} circuits={r.get('circuits')} "
      f"tokens={r.get('decode_tokens')} wall_us={r.get('wall_us')} "
      f"swap={[(x.get('swap_plan_bytes'), x.get('swap_in_bytes'), x.get('topups')) for x in r.get('stages', [])]}",
      flush=True)
if profile:
    for x in r.get("stages", []):
        kern = x.get("kernels", {})
        busy = sum(v["ms"] for k, v in kern.items() if isinstance(v, dict) and k != "swap_wait")
        sw = kern.get("swap_wait", {})
        print(f"rank {rank} kernels_ms={busy:.1f} swap_wait_ms={sw.get('ms', 0):.2f} "
              f"swap_waits={sw.get('n', 0)}", flush=True)
if st != 0:  # exit now: torchrun then stops the peers (a barrier would wait on them forever)
    os._exit(1)
if rank == world - 1 and r.get("tokens"):
    json.dump(r["tokens"], open(os.path.join(ROOT, "gpurun_out", f"nccl_tokens_{world}.json"), "w"))
dist.barrier()
lib.ds_session_destroy(h)
