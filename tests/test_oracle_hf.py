"""Pins the stage-forward oracle (oracle/llama_ref.c) against the canonical Llama implementation:
Hugging Face `transformers` LlamaForCausalLM in bf16 on CPU (the paper's serving system runs
PyTorch Llama-3 models; the reference simulator has no arithmetic). Same
counter-hash weights (canonical layout, RMSNorm gains 1), same prompt tokens, whole tiny model
(4 layers, GQA 4:2, RoPE theta 5e5): logits within the bf16 tolerance used for the GPU path
(|d| <= 0.08 + 0.02 |x|) and identical greedy tokens wherever the top-2 margin exceeds 0.16.
Test-only: transformers / torch CPU are checkers here, never the product."""
import ctypes as C

import numpy as np
import pytest

torch = pytest.importorskip("torch")
transformers = pytest.importorskip("transformers")

from paper_2501_14784_b200 import pipeline as pl  # noqa: E402
from paper_2501_14784_b200.bf16 import from_bf16, to_bf16  # noqa: E402

PHI = np.uint64(0x9E3779B97F4A7C15)
MIX_C = np.uint64(0xD1B54A32D192ED03)


def _mix64(z):
    z = (z ^ (z >> np.uint64(30))) * np.uint64(0xBF58476D1CE4E5B9)
    z = (z ^ (z >> np.uint64(27))) * np.uint64(0x94D049BB133111EB)
    return z ^ (z >> np.uint64(31))


def _weights(seed, tensor_id, rows, cols, scale):
    """lr_weight (oracle/llama_ref.c:49-53) for a whole [rows, cols] tensor, as float32 (the
    oracle's own OpenMP filler for big tensors; the numpy restatement below for small ones, which
    also cross-checks the filler)."""
    if rows * cols >= (1 << 22):
        import oracle
        lib = oracle.LlamaRef().lib
        lib.lr_fill_weights.argtypes = [C.c_uint64, C.c_uint64, C.c_int64, C.c_float, C.c_void_p]
        out = np.empty((rows, cols), dtype=np.float32)
        lib.lr_fill_weights(seed, tensor_id, rows * cols, scale, out.ctypes.data)
        return out
    idx = np.arange(rows * cols, dtype=np.uint64)
    with np.errstate(over="ignore"):
        h = _mix64(np.uint64(seed) + np.uint64(tensor_id) * PHI + idx * MIX_C)
    u = (h >> np.uint64(40)).astype(np.float32) * np.float32(1.0 / 16777216.0)
    v = (np.float32(2.0) * u - np.float32(1.0)) * np.float32(scale)
    return from_bf16(to_bf16(v)).reshape(rows, cols)


def _hf_model(dims, seed):
    d, nh, nkv, dh, ffn, V, L = (dims["d_model"], dims["n_heads"], dims["n_kv_heads"], dims["d_head"],
                                 dims["ffn"], dims["vocab"], dims["n_layers"])
    cfg = transformers.LlamaConfig(vocab_size=V, hidden_size=d, intermediate_size=ffn,
                                   num_hidden_layers=L, num_attention_heads=nh,
                                   num_key_value_heads=nkv, head_dim=dh,
                                   max_position_embeddings=dims["max_seq_len"],
                                   rope_theta=dims["rope_theta"], rms_norm_eps=dims["norm_eps"],
                                   tie_word_embeddings=False, attention_bias=False, mlp_bias=False)
    model = transformers.LlamaForCausalLM(cfg).eval()
    qd, kvd = nh * dh, nkv * dh
    sd, sq, sf = np.sqrt(3.0 / d), np.sqrt(3.0 / qd), np.sqrt(3.0 / ffn)
    t = lambda a: torch.from_numpy(np.ascontiguousarray(a))  # noqa: E731
    with torch.no_grad():
        model.model.embed_tokens.weight.copy_(t(_weights(seed, 1 << 20, V, d, 1.0)))
        model.lm_head.weight.copy_(t(_weights(seed, (1 << 20) + 1, V, d, sd)))
        model.model.norm.weight.fill_(1.0)
        for i, layer in enumerate(model.model.layers):
            base = i * 16
            a = layer.self_attn
            a.q_proj.weight.copy_(t(_weights(seed, base + 1, qd, d, sd)))
            a.k_proj.weight.copy_(t(_weights(seed, base + 2, kvd, d, sd)))
            a.v_proj.weight.copy_(t(_weights(seed, base + 3, kvd, d, sd)))
            a.o_proj.weight.copy_(t(_weights(seed, base + 4, d, qd, sq)))
            m = layer.mlp
            m.gate_proj.weight.copy_(t(_weights(seed, base + 6, ffn, d, sd)))
            m.up_proj.weight.copy_(t(_weights(seed, base + 7, ffn, d, sd)))
            m.down_proj.weight.copy_(t(_weights(seed, base + 8, d, ffn, sf)))
            layer.input_layernorm.weight.fill_(1.0)
            layer.post_attention_layernorm.weight.fill_(1.0)
    return model.to(torch.bfloat16)


def _oracle_logits(dims, seed, req, n_tok):
    import oracle
    from paper_2501_14784_b200._native import Row
    lr = oracle.LlamaRef()
    m = oracle.LrModel(**dims)
    st = lr.lib.lr_stage_create(C.byref(m), 0, dims["n_layers"], 1, 1, seed, 4)
    try:
        rows = (Row * 1)(Row(slot=0, pos=0, n_tok=n_tok, need_logits=1, is_decode=0, reserved=0,
                             req_id=req))
        tok = np.array([lr.lib.lr_prompt_token(req, p) for p in range(n_tok)], dtype=np.int32)
        act = np.zeros((n_tok, dims["d_model"]), dtype=np.float32)
        lg = np.zeros((1, dims["vocab"]), dtype=np.float32)
        ids = np.zeros(1, dtype=np.int32)
        rc = lr.lib.lr_stage_step(st, 0, 4, rows, 1, tok.ctypes.data, None, act.ctypes.data,
                                  lg.ctypes.data, ids.ctypes.data)
        assert rc == 0
        return tok, lg[0]
    finally:
        lr.lib.lr_stage_destroy(st)


@pytest.mark.parametrize("req,n_tok", [(7, 24), (11, 9)])
def test_oracle_matches_hf_llama(req, n_tok):
    dims = dict(pl.MODEL_DIMS["tiny-llama"])
    seed = pl.WEIGHT_SEED
    tok, ours = _oracle_logits(dims, seed, req, n_tok)
    model = _hf_model(dims, seed)
    with torch.no_grad():
        hf = model(torch.from_numpy(tok.astype(np.int64))[None, :]).logits[0, -1].float().numpy()
    err = np.abs(ours - hf)
    assert np.all(err <= 0.08 + 0.02 * np.abs(hf)), float(err.max())
    top = np.sort(hf)[-2:]
    if top[1] - top[0] > 0.16:
        assert int(np.argmax(ours)) == int(np.argmax(hf))


def test_weight_filler_matches_numpy_restatement():
    import oracle
    lib = oracle.LlamaRef().lib
    lib.lr_fill_weights.argtypes = [C.c_uint64, C.c_uint64, C.c_int64, C.c_float, C.c_void_p]
    out = np.empty((64, 96), dtype=np.float32)
    lib.lr_fill_weights(pl.WEIGHT_SEED, 37, out.size, 0.05, out.ctypes.data)
    assert np.array_equal(out, _weights(pl.WEIGHT_SEED, 37, 64, 96, 0.05))


def test_oracle_matches_hf_llama_at_8b_dims():
    """The same pin at the real Llama-3-8B dimensions (d 4096, 32 query / 8 KV heads of 128,
    ffn 14336, vocab 128256, RoPE theta 5e5), two layers: the GQA 4:1 head mapping, the 128-wide
    rotary halves and the LM head over the full vocabulary are checked, not just the tiny model's."""
    dims = dict(pl.MODEL_DIMS["llama3-8b"], n_layers=2)
    seed = pl.WEIGHT_SEED
    tok, ours = _oracle_logits(dims, seed, 21, 12)
    model = _hf_model(dims, seed)
    with torch.no_grad():
        hf = model(torch.from_numpy(tok.astype(np.int64))[None, :]).logits[0, -1].float().numpy()
    del model
    err = np.abs(ours - hf)
    assert np.all(err <= 0.08 + 0.02 * np.abs(hf)), float(err.max())
    top = np.sort(hf)[-2:]
    if top[1] - top[0] > 0.16:
        assert int(np.argmax(ours)) == int(np.argmax(hf))


def test_oracle_matches_hf_llama_at_70b_dims():
    """The pin at the Llama-3-70B dimensions (d 8192, 64 query / 8 KV heads of 128 = GQA 8:1, ffn
    28672, vocab 128256), one layer: the 8:1 head mapping the 70B stages use, checked against
    transformers on the same counter-hash weights."""
    dims = dict(pl.MODEL_DIMS["llama3-70b-bf16"], n_layers=1)
    seed = pl.WEIGHT_SEED
    tok, ours = _oracle_logits(dims, seed, 5, 10)
    model = _hf_model(dims, seed)
    with torch.no_grad():
        hf = model(torch.from_numpy(tok.astype(np.int64))[None, :]).logits[0, -1].float().numpy()
    del model
    err = np.abs(ours - hf)
    assert np.all(err <= 0.08 + 0.02 * np.abs(hf)), float(err.max())
    top = np.sort(hf)[-2:]
    if top[1] - top[0] > 0.16:
        assert int(np.argmax(ours)) == int(np.argmax(hf))
