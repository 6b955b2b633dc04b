"""KV swap round trips (reference issue_swap_in, src/sim.cpp:328-353) keep the cache bit-exact.

ds_swap_in overlaps the eviction (D2H) with the refill (H2D) page by page: an H2D into a slot
page waits only for that page's eviction and for the D2H of the host page it reads. This test
runs the same rows on two stages with the same weights -- one holding every page locally, one
with a single local page per microbatch and the rest in host-backed global slots, swapped back
and forth -- and requires bit-identical activations from a prompt continuation whose attention
reads every swapped page.
"""
import ctypes as C

import pytest
import torch

from paper_2501_14784_b200 import _native as nat
from paper_2501_14784_b200 import pipeline as pl

pytestmark = pytest.mark.gpu

DIMS = pl.MODEL_DIMS["tiny-llama"]
LAYERS = 4
PAGE = 256 * LAYERS * 2 * DIMS["n_kv_heads"] * DIMS["d_head"] * 2
FILL = [(0, 600, 0), (1, 300, 10), (2, 520, 20)]  # (slot, prompt tokens, request id base)


def _rows(spec):
    return (nat.Row * len(spec))(*[nat.Row(slot=s, pos=p, n_tok=n, need_logits=0, is_decode=0,
                                           reserved=0, req_id=r) for s, p, n, r in spec])


def _run(swapping, cycles=5):
    md = pl.model_desc(DIMS)
    st = C.c_void_p()
    nat.check(nat.lib.ds_stage_create(0, C.byref(md), 0, LAYERS, 1, 0, 11, 2048, 4, C.byref(st)))
    try:
        if swapping:
            nat.check(nat.lib.ds_kv_create(st, PAGE, 2, PAGE, 12 * PAGE, 12 * PAGE))
        else:
            nat.check(nat.lib.ds_kv_create(st, PAGE, 2, 16 * PAGE, 0, 0))
        mi, mo = C.c_int64(), C.c_int64()
        moved = 0
        for mb in range(2):
            if swapping:
                nat.check(nat.lib.ds_swap_in(st, mb, mb if cycles < 0 else 0, 0, C.byref(mi),
                                             C.byref(mo)))
            spec = [(s, 0, n, r + mb) for s, n, r in FILL]
            nat.check(nat.lib.ds_stage_step(st, mb, _rows(spec), len(spec), None, None))
        if swapping:
            # slot 0 alternates between the microbatches (evict + refill every call), then mb 1
            # comes back into slot 1 next to mb 0
            for r in range(cycles):
                nat.check(nat.lib.ds_swap_in(st, r % 2, 0, 0, C.byref(mi), C.byref(mo)))
                moved += mi.value + mo.value
            if cycles >= 0:
                nat.check(nat.lib.ds_swap_in(st, cycles % 2, 1, 0, C.byref(mi), C.byref(mo)))
                moved += mi.value + mo.value
            for mb in range(2):
                res = C.c_int32()
                nat.check(nat.lib.ds_kv_resident(st, mb, C.byref(res)))
                assert res.value == 1
        outs = []
        for mb in (1, 0):
            spec = [(s, n, 8, r + mb) for s, n, r in FILL]
            T = sum(x[2] for x in spec)
            out = torch.empty(T, DIMS["d_model"], dtype=torch.bfloat16, device="cuda")
            nat.check(nat.lib.ds_stage_step(st, mb, _rows(spec), len(spec), None,
                                            C.c_void_p(out.data_ptr())))
            nat.check(nat.lib.ds_stage_sync(st))
            outs.append(out.clone())
        return outs, moved
    finally:
        nat.lib.ds_stage_destroy(st)


@pytest.mark.parametrize("cycles", [0, 1, 5])
def test_swap_round_trips_bit_exact(cycles):
    """cycles = 0: one plain swap-in of an evicted microbatch; its compute must also wait for
    the eviction of the slot pages it appends into (regression of the overlapped copies)."""
    torch.cuda.init()
    ref, _ = _run(False)
    got, moved = _run(True, cycles)
    assert moved > 0
    for a, b in zip(ref, got):
        assert torch.isfinite(a.float()).all()
        assert torch.equal(a, b)


def test_refill_after_release_waits_for_the_occupants_step():
    """the occupant of a global slot runs a step, then releases a slot-backed request
    (its pages go back to the slot's free list without an eviction copy), and another
    microbatch is swapped into that slot before anything syncs: the refill must wait for the
    occupant's step, so the refilled microbatch computes exactly as without swapping."""
    torch.cuda.init()
    ref, _ = _run(False)
    md = pl.model_desc(DIMS)
    st = C.c_void_p()
    nat.check(nat.lib.ds_stage_create(0, C.byref(md), 0, LAYERS, 1, 0, 11, 2048, 4, C.byref(st)))
    try:
        nat.check(nat.lib.ds_kv_create(st, PAGE, 2, PAGE, 12 * PAGE, 12 * PAGE))
        mi, mo = C.c_int64(), C.c_int64()
        for mb in (1, 0):  # mb 1 filled first and evicted when mb 0 takes slot 0
            nat.check(nat.lib.ds_swap_in(st, mb, 0, 0, C.byref(mi), C.byref(mo)))
            spec = [(s, 0, n, r + mb) for s, n, r in FILL]
            nat.check(nat.lib.ds_stage_step(st, mb, _rows(spec), len(spec), None, None))
        # mb 0: one more step, then its slot-backed request in slot 0 completes
        spec = [(0, 600, 8, 0)]
        nat.check(nat.lib.ds_stage_step(st, 0, _rows(spec), 1, None, None))
        nat.check(nat.lib.ds_kv_release(st, 0, 0))
        # mb 1 back into slot 0 (freed pages of mb 0 are refilled) with no sync in between
        nat.check(nat.lib.ds_swap_in(st, 1, 0, 0, C.byref(mi), C.byref(mo)))
        spec = [(s, n, 8, r + 1) for s, n, r in FILL]
        T = sum(x[2] for x in spec)
        out = torch.empty(T, DIMS["d_model"], dtype=torch.bfloat16, device="cuda")
        nat.check(nat.lib.ds_stage_step(st, 1, _rows(spec), len(spec), None, C.c_void_p(out.data_ptr())))
        nat.check(nat.lib.ds_stage_sync(st))
        assert torch.equal(out, ref[0])
        stats = (C.c_int64 * 4)()
        nat.check(nat.lib.ds_swap_stats(st, stats))
        assert stats[0] > 0  # mb 1's host pages came back through the slot
    finally:
        nat.lib.ds_stage_destroy(st)
