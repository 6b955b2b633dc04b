"""Stage-forward parity: the sm_100a path through the C ABI vs the CPU oracle (oracle/llama_ref.c).

Tolerance (bf16 storage, fp32 accumulation; differences come from accumulation order and
occasional one-ulp bf16 rounding flips that propagate through the layers):
  logits:      |gpu - cpu| <= 0.08 + 0.02 * |cpu|   (logits have O(1) scale; attention rounds the
               softmax numerators to bf16 for the tensor-core P.V, as FlashAttention does)
  activations: |gpu - cpu| <= 0.03 * max|cpu| per row
  greedy:      gpu argmax == oracle argmax wherever the oracle's top-2 margin > 0.16
"""
import numpy as np
import pytest

from stage_harness import Pair, greedy_ok, logits_ok, random_act

pytestmark = pytest.mark.gpu

LOGIT_MARGIN = 0.16


def _check_logits(o):
    ok, err = logits_ok(o["gpu_logits"], o["cpu_logits"])
    assert ok, f"max |dlogit| {err}"
    assert not greedy_ok(o["gpu_ids"], o["cpu_logits"], LOGIT_MARGIN)
    return err


def test_tiny_whole_model_circuits():
    p = Pair("tiny-llama", 0, 4, True, True, n_mb=2, max_slots=8)
    try:
        # circuit 1: two prompts completing, one long prompt chunk, one empty-prompt decode (BOS)
        errs = []
        o = p.step(0, [(0, 0, 5, 1, 0, 10), (1, 0, 1, 1, 0, 11), (2, 0, 37, 0, 0, 12),
                       (3, 0, 1, 1, 1, 13)])
        errs.append(_check_logits(o))
        # circuit on the other microbatch: a prompt crossing the 256-token page boundary
        o = p.step(1, [(0, 0, 270, 1, 0, 20), (1, 0, 3, 1, 0, 21)])
        errs.append(_check_logits(o))
        # circuit 2 of mb 0: decodes (teacher-forced) + prompt continuation across a page
        o = p.step(0, [(0, 5, 1, 1, 1, 10), (1, 1, 1, 1, 1, 11), (2, 37, 300, 1, 0, 12),
                       (3, 1, 1, 1, 1, 13)])
        errs.append(_check_logits(o))
        for k in range(6):
            o = p.step(0, [(0, 6 + k, 1, 1, 1, 10), (1, 2 + k, 1, 1, 1, 11),
                           (2, 337 + k, 1, 1, 1, 12), (3, 2 + k, 1, 1, 1, 13)])
            errs.append(_check_logits(o))
            o = p.step(1, [(0, 270 + k, 1, 1, 1, 20), (1, 3 + k, 1, 1, 1, 21)])
            errs.append(_check_logits(o))
        # slot reuse: a new request in slot 1 of mb 0 resets its pages
        o = p.step(0, [(1, 0, 9, 1, 0, 99), (2, 343, 1, 1, 1, 12)])
        errs.append(_check_logits(o))
        print("tiny max |dlogit| per circuit:", [round(e, 4) for e in errs])
    finally:
        p.close()


def test_tiny_two_stage_activations_and_logits():
    a = Pair("tiny-llama", 0, 2, True, False, n_mb=1)
    b = Pair("tiny-llama", 2, 4, False, True, n_mb=1)
    try:
        rows = [(0, 0, 20, 1, 0, 5), (1, 0, 1, 1, 1, 6)]
        oa = a.step(0, rows)
        err = np.abs(oa["gpu_act"] - oa["cpu_act"]).max(axis=1)
        assert np.all(err <= 0.03 * np.abs(oa["cpu_act"]).max(axis=1)), err
        ob = b.step(0, rows, act_in=oa["cpu_act"])
        _check_logits(ob)
        a.last_tok = b.last_tok
        rows = [(0, 20, 1, 1, 1, 5), (1, 1, 1, 1, 1, 6)]
        oa = a.step(0, rows, ids_in=ob["gpu_ids"])
        ob = b.step(0, rows, act_in=oa["cpu_act"])
        _check_logits(ob)
    finally:
        a.close()
        b.close()


def test_llama8b_dims_first_stage_activations():
    # 2 real Llama-3-8B layers (d 4096, GQA 32:8, d_head 128, ffn 14336) as a first stage
    p = Pair("llama3-8b", 0, 2, True, False, n_mb=1, max_slots=4, pages_per_mb=8)
    try:
        for rows in ([(0, 0, 33, 1, 0, 1), (1, 0, 1, 1, 1, 2), (2, 0, 260, 1, 0, 3)],
                     [(1, 1, 1, 1, 1, 2), (0, 33, 4, 1, 0, 1)]):
            ids = None
            if rows[0][4]:  # previous circuit sampled rows: slots 0, 1, 2
                p.last_tok[(0, 1)] = 1234
                ids = np.array([111, 1234, 222], dtype=np.int32)
            o = p.step(0, rows, ids_in=ids)
            err = np.abs(o["gpu_act"] - o["cpu_act"]).max(axis=1)
            scale = np.abs(o["cpu_act"]).max(axis=1)
            assert np.all(err <= 0.03 * scale), (err / scale).max()
    finally:
        p.close()


def test_llama8b_dims_last_stage_logits():
    p = Pair("llama3-8b", 31, 32, False, True, n_mb=1, max_slots=4, pages_per_mb=8)
    try:
        rows = [(0, 0, 17, 1, 0, 1), (1, 0, 1, 1, 1, 2), (2, 0, 300, 1, 0, 3)]
        o = p.step(0, rows, act_in=random_act(318, 4096, 7))
        _check_logits(o)
        rows = [(0, 17, 1, 1, 1, 1), (1, 1, 1, 1, 1, 2), (2, 300, 1, 1, 1, 3)]
        o = p.step(0, rows, act_in=random_act(3, 4096, 8))
        _check_logits(o)
    finally:
        p.close()


def test_llama70b_dims_first_and_last_stage():
    # Llama-3-70B dims (d 8192, GQA 64:8 -> 8 query heads per KV head, ffn 28672): one layer as a
    # first stage and the last layer + LM head as a last stage (BASELINE configs[3] shapes)
    a = Pair("llama3-70b-bf16", 0, 1, True, False, n_mb=1, max_slots=4, pages_per_mb=8)
    try:
        rows = [(0, 0, 40, 1, 0, 1), (1, 0, 1, 1, 1, 2), (2, 0, 270, 1, 0, 3)]
        o = a.step(0, rows)
        err = np.abs(o["gpu_act"] - o["cpu_act"]).max(axis=1)
        assert np.all(err <= 0.03 * np.abs(o["cpu_act"]).max(axis=1)), err
        rows = [(0, 40, 1, 1, 1, 1), (1, 1, 1, 1, 1, 2), (2, 270, 1, 1, 1, 3)]
        for slot, tok in enumerate((5, 6, 7)):  # the previous circuit's samples, in row order
            a.last_tok[(0, slot)] = tok
        o = a.step(0, rows, ids_in=np.array([5, 6, 7], dtype=np.int32))
        err = np.abs(o["gpu_act"] - o["cpu_act"]).max(axis=1)
        assert np.all(err <= 0.03 * np.abs(o["cpu_act"]).max(axis=1)), err
    finally:
        a.close()
    b = Pair("llama3-70b-bf16", 79, 80, False, True, n_mb=1, max_slots=4, pages_per_mb=8)
    try:
        rows = [(0, 0, 17, 1, 0, 1), (1, 0, 1, 1, 1, 2), (2, 0, 300, 1, 0, 3)]
        _check_logits(b.step(0, rows, act_in=random_act(318, 8192, 9)))
        rows = [(0, 17, 1, 1, 1, 1), (1, 1, 1, 1, 1, 2), (2, 300, 1, 1, 1, 3)]
        _check_logits(b.step(0, rows, act_in=random_act(3, 8192, 10)))
    finally:
        b.close()


def test_llama8b_dims_long_prefill_chunk():
    # a 700-row prefill circuit (prefill_chunk > 512): 256-token GEMM blocks in token-block-
    # fastest order, token-split q/k/v and o, prompt attention over three KV pages
    p = Pair("llama3-8b", 0, 2, True, False, max_rows=768, n_mb=1, max_slots=4, pages_per_mb=8)
    try:
        rows = [(0, 0, 600, 1, 0, 1), (1, 0, 100, 1, 0, 2)]
        o = p.step(0, rows)
        err = np.abs(o["gpu_act"] - o["cpu_act"]).max(axis=1)
        assert np.all(err <= 0.03 * np.abs(o["cpu_act"]).max(axis=1)), (err / np.abs(o["cpu_act"]).max(axis=1)).max()
    finally:
        p.close()
