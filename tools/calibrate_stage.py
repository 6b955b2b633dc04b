#!/usr/bin/env python3
"""Measured stage-time points for the calibration CSV (reference format
perf_model.cpp:44-83): one stage of `--layers` layers (embedding + LM head when it is the whole
model) on one B200, timed on synthetic circuits of T rows:

  * decode circuits (T <= 512): T decode rows at context --ctx (the paper's Table 1 shape,
    "decoding with same prefix"), every row sampling a token;
  * prefill circuits (T > 512): whole --prompt-token prompts packed into the chunk (the
    swap-forcing workloads: 3840-token prompts, prefill_chunk 16384), the last one partial.

Median of --reps steps after 2 warm-ups, from empty KV pools. Prints CSV rows (batch_size,
total_time_ms) and writes --out JSON.
"""
import argparse
import ctypes as C
import json
import os
import statistics
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2501_14784_b200 import _native as nat  # noqa: E402
from paper_2501_14784_b200 import pipeline as pl  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--model", default="llama3-8b")
    ap.add_argument("--layers", type=int, default=32)
    ap.add_argument("--first-layer", type=int, default=0)
    ap.add_argument("--ctx", type=int, default=512)
    ap.add_argument("--prompt", type=int, default=3840)
    ap.add_argument("--decode", default="1,2,4,8,16,32,64,96,128,192,256,320,384,448,512")
    ap.add_argument("--prefill", default="1024,2048,3840,7680,11520,16384")
    ap.add_argument("--reps", type=int, default=5)
    ap.add_argument("--out", default=os.path.join(ROOT, "gpurun_out", "calibration.json"))
    a = ap.parse_args()
    dims = pl.MODEL_DIMS[a.model]
    lb, le = a.first_layer, a.first_layer + a.layers
    first, last = lb == 0, le == dims["n_layers"]
    dec = [int(x) for x in a.decode.split(",") if x]
    pre = [int(x) for x in a.prefill.split(",") if x]
    max_rows = max(dec + pre)
    slots = max(max(dec, default=1), max(pre, default=0) // a.prompt + 2)
    md = pl.model_desc(dims)
    st = C.c_void_p()
    nat.check(nat.lib.ds_stage_create(0, C.byref(md), lb, le, int(first), int(last), pl.WEIGHT_SEED,
                                      (max_rows + 15) // 16 * 16, slots, C.byref(st)))
    page = 256 * a.layers * 2 * dims["n_kv_heads"] * dims["d_head"] * 2
    need_pages = max(max(dec, default=0) * ((a.ctx + 1 + 255) // 256), max(pre, default=0) // 256 + slots)
    nat.check(nat.lib.ds_kv_create(st, page, 1, need_pages * page, 0, 0))
    act = C.c_void_p()
    nat.check(nat.lib.ds_dbg_alloc(0, max_rows * dims["d_model"] * 2, C.byref(act)))
    ids = C.c_void_p()
    nat.check(nat.lib.ds_dbg_alloc(0, max_rows * 4, C.byref(ids)))
    out = []

    def timed(rows):
        arr = (nat.Row * len(rows))(*[nat.Row(slot=r[0], pos=r[1], n_tok=r[2], need_logits=r[3],
                                              is_decode=r[4], reserved=0, req_id=r[5]) for r in rows])
        ts = []
        for k in range(a.reps + 2):
            nat.check(nat.lib.ds_kv_reset(st))
            t0 = time.perf_counter()
            nat.check(nat.lib.ds_stage_step(st, 0, arr, len(rows), None if first else act,
                                            ids if last else None))
            nat.check(nat.lib.ds_stage_sync(st))
            if k >= 2:
                ts.append((time.perf_counter() - t0) * 1e3)
        return statistics.median(ts)

    try:
        for T in dec:  # T decode rows at context ctx
            ms = timed([(i, a.ctx, 1, 1, 1, 1000 + i) for i in range(T)])
            out.append((T, ms))
            print(f"{T},{ms:.3f}", flush=True)
        for T in pre:  # whole prompts packed into a T-row chunk
            rows, left, i = [], T, 0
            while left > 0:
                n = min(a.prompt, left)
                rows.append((i, 0, n, 1 if n == a.prompt else 0, 0, 5000 + i))
                left -= n
                i += 1
            ms = timed(rows)
            out.append((T, ms))
            print(f"{T},{ms:.3f}", flush=True)
    finally:
        nat.lib.ds_dbg_free(act)
        nat.lib.ds_dbg_free(ids)
        nat.lib.ds_stage_destroy(st)
    json.dump({"model": a.model, "layers": a.layers, "ctx": a.ctx, "prompt": a.prompt, "points": out},
              open(a.out, "w"), indent=1)


if __name__ == "__main__":
    main()
