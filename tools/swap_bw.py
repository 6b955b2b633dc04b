"""KV swap bandwidth on one B200: ds_swap_in (C ABI) against the measured host link.

north_star (3): the swap of reference issue_swap_in (src/sim.cpp:328-353) runs as pinned
cudaMemcpyAsync page copies on the stage's D2H / H2D copy streams; its evidence is swap GB/s
against the host link measured on the same box. This tool measures
  * the host link: pinned <-> device copies of 1 GiB (H2D alone, D2H alone, both directions
    concurrently on two streams), best of 5, host-timed around a device synchronize;
  * ds_swap_in at the Llama-3-8B 4-stage page size (8 layers, 8,388,608 B pages): two
    microbatches whose KV lives in a host-backed global slot are swapped through one slot in
    turn, so every call evicts the occupant (D2H) and brings the target in (H2D). The H2D into
    a slot page waits only for that page's eviction, so the two directions overlap and the
    bound is the concurrent (bidirectional) host-link rate. Timed on the host around a device
    synchronize (each call moves ~1.6 GB).
Prints one JSON line; `python tools/swap_bw.py > profiles/r01_swap_bw.json` under gpurun.
"""
import ctypes as C
import argparse
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402

from paper_2501_14784_b200 import _native as nat  # noqa: E402
from paper_2501_14784_b200 import pipeline as pl  # noqa: E402


def host_link(nbytes=1 << 30, reps=5):
    h = torch.empty(nbytes, dtype=torch.uint8, pin_memory=True)
    h2 = torch.empty(nbytes, dtype=torch.uint8, pin_memory=True)
    d = torch.empty(nbytes, dtype=torch.uint8, device="cuda")
    d2 = torch.empty(nbytes, dtype=torch.uint8, device="cuda")
    s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()

    def timed(fn):
        fn()
        torch.cuda.synchronize()
        best = 1e9
        for _ in range(reps):
            t0 = time.perf_counter()
            fn()
            torch.cuda.synchronize()
            best = min(best, time.perf_counter() - t0)
        return best

    def h2d():
        with torch.cuda.stream(s1):
            d.copy_(h, non_blocking=True)

    def d2h():
        with torch.cuda.stream(s2):
            h2.copy_(d2, non_blocking=True)

    def both():
        h2d()
        d2h()

    th, td, tb = timed(h2d), timed(d2h), timed(both)
    return {"bytes": nbytes, "h2d_gbs": nbytes / th / 1e9, "d2h_gbs": nbytes / td / 1e9,
            "bidir_gbs": 2 * nbytes / tb / 1e9}


def swap(model="llama3-8b", n_layers=8, tokens_per_mb=24 * 1024, rounds=6):
    dims = dict(pl.MODEL_DIMS[model])
    md = pl.model_desc(dims)
    st = C.c_void_p()
    max_rows = 4096
    nat.check(nat.lib.ds_stage_create(0, C.byref(md), 0, n_layers, 1, 0, 7, max_rows, 8, C.byref(st)))
    page = 256 * n_layers * 2 * dims["n_kv_heads"] * dims["d_head"] * 2
    pages = tokens_per_mb // 256
    # 1 local page per microbatch; the rest lives in the global slot and the pinned host backing
    nat.check(nat.lib.ds_kv_create(st, page, 2, page, (pages + 1) * page, (pages + 1) * page))
    mi, mo = C.c_int64(), C.c_int64()
    req = 0
    for mb in range(2):
        nat.check(nat.lib.ds_swap_in(st, mb, 0, 0, C.byref(mi), C.byref(mo)))
        for slot in range(tokens_per_mb // max_rows):
            rows = (nat.Row * 1)(nat.Row(slot=slot, pos=0, n_tok=max_rows, need_logits=0,
                                         is_decode=0, reserved=0, req_id=req))
            req += 1
            nat.check(nat.lib.ds_stage_step(st, mb, rows, 1, None, None))
        nat.check(nat.lib.ds_stage_sync(st))
    torch.cuda.synchronize()
    res = []
    for r in range(rounds + 1):
        mb = r % 2  # the microbatch not in slot 0 (mb 1 holds it after the fill)
        t0 = time.perf_counter()
        nat.check(nat.lib.ds_swap_in(st, mb, 0, 0, C.byref(mi), C.byref(mo)))
        torch.cuda.synchronize()
        dt = time.perf_counter() - t0
        if r > 0:
            res.append((mi.value, mo.value, dt))
    nat.lib.ds_stage_destroy(st)
    moved = sum(a + b for a, b, _ in res)
    t = sum(x for _, _, x in res)
    return {"model": model, "layers": n_layers, "page_bytes": page, "pages_per_mb": pages, "calls": len(res),
            "in_bytes_per_call": res[0][0], "out_bytes_per_call": res[0][1],
            "ms_per_call": 1e3 * t / len(res), "gbs": moved / t / 1e9}


def main():
    torch.cuda.init()
    link = host_link()
    # default: the 8B 4-stage page; "--model llama3-70b-bf16 --layers 10" = the 70B 8-stage page
    ap = argparse.ArgumentParser()
    ap.add_argument("--model", default=None)
    ap.add_argument("--layers", type=int, default=None)
    a = ap.parse_args()
    if (a.model is None) != (a.layers is None):
        sys.exit("swap_bw.py: give both --model and --layers, or neither")
    sw = swap(a.model, a.layers) if a.model else swap()
    # eviction and refill overlap page by page: the bound is both directions at once
    bound_s = (sw["out_bytes_per_call"] + sw["in_bytes_per_call"]) / (link["bidir_gbs"] * 1e9)
    sw["bound_ms_per_call"] = 1e3 * bound_s
    sw["frac_of_host_link"] = sw["bound_ms_per_call"] / sw["ms_per_call"]
    print(json.dumps({"host_link": link, "swap_in": sw,
                      "device": torch.cuda.get_device_name(0)}))


if __name__ == "__main__":
    main()
