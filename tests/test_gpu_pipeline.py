"""Whole-pipeline GPU runs through ds_gpu_run_config (replay of the integer schedule):
tiny 2-stage (BASELINE configs[0]) with and without KV swap, checked against the CPU oracle
(teacher-forced greedy agreement) and against the schedule's integer contract."""
import json
import os

import numpy as np
import pytest

from paper_2501_14784_b200 import pipeline as pl

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
CONFIGS = os.path.join(ROOT, "configs")


def _cfg(name, **wl):
    cfg = json.load(open(os.path.join(CONFIGS, name)))
    cfg["workload"].update(wl)
    return json.dumps(cfg)


def _oracle_tokens(txt, n_circ, gpu_tokens):
    """Replays the first n_circ circuits on the CPU oracle (both stages), teacher-forced with
    the GPU's sampled ids; returns per circuit the oracle logits of the sampled rows."""
    import ctypes as C

    import oracle
    from paper_2501_14784_b200._native import Row
    sched = pl.schedule_config(txt, CONFIGS, max_circuits=n_circ)
    plan = json.loads(pl.plan_config(txt, CONFIGS))
    dims = pl.MODEL_DIMS["tiny-llama"]
    lr = oracle.LlamaRef()
    m = oracle.LrModel(**dims)
    S = len(plan["stages"])
    B = plan["stages"][0]["batch_size_per_microbatch"]
    NB = plan["n_microbatches"]
    st = [lr.lib.lr_stage_create(C.byref(m), s["layer_begin"], s["layer_end"], int(i == 0),
                                 int(i == S - 1), pl.WEIGHT_SEED, NB * B)
          for i, s in enumerate(plan["stages"])]
    last = {}
    out = []
    for ci, c in enumerate(sched["circuits"]):
        rows = c["rows"]
        arr = (Row * len(rows))(*[Row(slot=r[0], pos=r[1], n_tok=r[2], need_logits=r[3],
                                      is_decode=r[4], reserved=0, req_id=r[5]) for r in rows])
        toks = []
        for r in rows:
            for j in range(r[2]):
                pos = r[1] + j
                toks.append((128000 if pos == 0 else last[(c["mb"], r[0])]) if r[4]
                            else lr.lib.lr_prompt_token(r[5], pos))
        T = sum(r[2] for r in rows)
        R = sum(r[3] for r in rows)
        tok = np.array(toks, dtype=np.int32)
        act = np.zeros((T, dims["d_model"]), dtype=np.float32)
        act2 = np.zeros_like(act)
        lg = np.zeros((max(R, 1), dims["vocab"]), dtype=np.float32)
        ids = np.zeros(max(R, 1), dtype=np.int32)
        for i in range(S):
            src = act if i % 2 == 0 else act2
            dst = act2 if i % 2 == 0 else act
            rc = lr.lib.lr_stage_step(st[i], c["mb"], B, arr, len(rows), tok.ctypes.data,
                                      src.ctypes.data if i else None, dst.ctypes.data,
                                      lg.ctypes.data if i == S - 1 else None, ids.ctypes.data)
            assert rc == 0
        k = 0
        for r in rows:
            if r[3]:
                last[(c["mb"], r[0])] = gpu_tokens[ci][k]
                k += 1
        out.append(lg[:R])
    for s in st:
        lr.lib.lr_stage_destroy(s)
    return sched, out


@pytest.mark.parametrize("name", ["tiny_2stage.json", "tiny_2stage_swap.json"])
def test_tiny_pipeline_matches_oracle(name):
    txt = _cfg(name, bench_duration_s=30, warmup_s=1)
    n = 120
    r = pl.gpu_run_config(txt, CONFIGS, collect_tokens=True, max_circuits=n, real_delay=False)
    assert r["error"] == "" and r["circuits"] == n
    sched, logits = _oracle_tokens(txt, n, r["tokens"])
    assert sum(c["n_decode"] for c in sched["circuits"]) == r["decode_tokens"]
    checked = mism = 0
    for ci in range(n):
        for k, row in enumerate(logits[ci]):
            top = np.sort(row)[-2:]
            if top[1] - top[0] > 0.16:
                checked += 1
                mism += int(np.argmax(row) != r["tokens"][ci][k])
    assert checked > 0 and mism == 0, (checked, mism)
    if "swap" in name:
        st = r["stages"]
        assert sum(s["swap_in_bytes"] for s in st) > 0  # the swap path really moved pages
        assert sum(s["swap_plan_bytes"] for s in st) > 0


def test_tiny_pipeline_real_delay_and_trace_timing(tmp_path):
    txt = _cfg("tiny_2stage.json", bench_duration_s=30, warmup_s=0)
    tr = str(tmp_path / "hw.trace")
    res = pl.run(txt, CONFIGS, max_circuits=40, real_delay=True, trace_path=tr)
    r = res["gpu"]
    assert r["error"] == ""
    # 40 circuits over 8 microbatches at 10 ms per hop: >= 5 ring rounds * 2 hops * 10 ms
    assert r["wall_us"] >= 5 * 2 * 10000
    # every hop arrival in the real-clock trace honours send + latency + serialisation (the
    # reference's transfer-causality rule, sim.cpp:656-669), measured on the host clock
    n = 0
    for line in open(tr):
        f = dict(x.split("=", 1) for x in line.split())
        if f["kind"] == "TransferArrive" and int(f["t"]) > 0:
            n += 1
            assert int(f["t"]) >= int(f["a"]) + 10000 + (int(f["b"]) * 10**6 + 1250000000 - 1) // 1250000000
    assert n > 0
