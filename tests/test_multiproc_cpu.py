"""N>1 host logic on CPU (gloo, world_size 2): every rank derives the identical schedule from the
config (the NCCL hops pair sends and receives purely from it, executor.cpp receiver()), the
NCCL unique ids travel through the launcher's store, and each link's send sequence (producer
compute order, sizes) equals the receive sequence the consumer will post."""
import hashlib
import json
import os
import socket

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _hop_sequence(sched, from_stage, to_stage, d_model):
    seq = []
    for op in sched["ops"][from_stage]:
        if op[0] != 0:
            continue
        c = sched["circuits"][op[3]]
        # the ids hop always carries >= 1 int32: stage 0 times every circuit end (trace arrival
        # of woken microbatches, reference wake_parked sim.cpp:277-294)
        nbytes = (max(sum(r[3] for r in c["rows"]), 1) * 4 if to_stage == 0
                  else c["eff_batch"] * d_model * 2)
        if nbytes:
            seq.append((op[3], c["mb"], nbytes))
    return seq


def _worker(rank, world, port, q):
    import sys
    sys.path.insert(0, ROOT)
    import ctypes as C

    import torch.distributed as dist

    from paper_2501_14784_b200 import pipeline as pl
    from paper_2501_14784_b200._native import check, lib
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        ids = [None]
        if rank == 0:
            buf = (C.c_uint8 * 128)()
            check(lib.ds_nccl_unique_id(buf))
            ids = [bytes(buf) * world]
        dist.broadcast_object_list(ids, src=0)
        cdir = os.path.join(ROOT, "configs")
        txt = open(os.path.join(cdir, "tiny_2stage_swap.json")).read()
        sched = pl.schedule_config(txt, cdir, max_circuits=500)
        h = hashlib.sha256(json.dumps(sched, sort_keys=True).encode()).hexdigest()
        # what this rank sends (its compute order) and what it will receive (previous stage's)
        sends = _hop_sequence(sched, rank, (rank + 1) % world, 256)
        recvs = _hop_sequence(sched, (rank - 1) % world, rank, 256)
        out = [None] * world
        dist.all_gather_object(out, {"hash": h, "ids": ids[0][:16], "sends": sends, "recvs": recvs})
        q.put((rank, out))
    finally:
        dist.destroy_process_group()


def test_two_rank_schedule_and_link_pairing():
    import torch.multiprocessing as mp
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = dict(q.get(timeout=300) for _ in procs)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    view = res[0]
    assert view[0]["hash"] == view[1]["hash"]
    assert view[0]["ids"] == view[1]["ids"]
    # link 0 -> 1: rank 0's sends are exactly rank 1's receives; link 1 -> 0 likewise (ids)
    assert view[0]["sends"] == view[1]["recvs"] and len(view[0]["sends"]) > 0
    assert view[1]["sends"] == view[0]["recvs"] and len(view[1]["sends"]) > 0
    # the ids hop carries one int32 per sampled row
    assert all(b % 4 == 0 for _, _, b in view[1]["sends"])
