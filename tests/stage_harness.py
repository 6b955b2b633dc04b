"""Drives one GPU stage (C ABI) and the CPU oracle stage (oracle/llama_ref.c) on identical rows.

Teacher forcing: decode rows take as input the token the GPU sampled for that slot in the
microbatch's previous circuit; the oracle is fed the same token, so logits stay comparable even
where greedy choices of a random-init model are near-ties."""
import ctypes as C

import numpy as np

from paper_2501_14784_b200 import _native as nat
from paper_2501_14784_b200 import pipeline as pl
from paper_2501_14784_b200.bf16 import round_bf16

BOS = 128000


class Pair:
    def __init__(self, model, lb, le, first, last, max_rows=512, max_slots=8, n_mb=2,
                 pages_per_mb=64, seed=pl.WEIGHT_SEED):
        import oracle
        self.dims = pl.MODEL_DIMS[model] if isinstance(model, str) else model
        self.first, self.last = first, last
        self.max_slots = max_slots
        md = pl.model_desc(self.dims)
        self.st = C.c_void_p()
        nat.check(nat.lib.ds_stage_create(0, C.byref(md), lb, le, int(first), int(last), seed,
                                          max_rows, max_slots, C.byref(self.st)))
        d = self.dims
        page = 256 * (le - lb) * 2 * d["n_kv_heads"] * d["d_head"] * 2
        nat.check(nat.lib.ds_kv_create(self.st, page, n_mb, pages_per_mb * page, 0, 0))
        self.lr = oracle.LlamaRef()
        m = oracle.LrModel(**d)
        self.cs = self.lr.lib.lr_stage_create(C.byref(m), lb, le, int(first), int(last), seed,
                                              n_mb * max_slots)
        self.last_tok = {}
        self.d_act = C.c_void_p()
        nat.check(nat.lib.ds_dbg_alloc(0, max_rows * d["d_model"] * 2, C.byref(self.d_act)))
        self.d_ids = C.c_void_p()
        nat.check(nat.lib.ds_dbg_alloc(0, max_rows * 4, C.byref(self.d_ids)))

    def close(self):
        nat.lib.ds_dbg_free(self.d_act)
        nat.lib.ds_dbg_free(self.d_ids)
        nat.lib.ds_stage_destroy(self.st)
        self.lr.lib.lr_stage_destroy(self.cs)

    def step(self, mb, rows, act_in=None, ids_in=None):
        """rows: (slot, pos, n_tok, need_logits, is_decode, req). Returns dict with GPU/CPU
        activations or logits/ids."""
        d = self.dims["d_model"]
        V = self.dims["vocab"]
        R = sum(r[3] for r in rows)
        T = sum(r[2] for r in rows)
        arr = (nat.Row * len(rows))(*[nat.Row(slot=r[0], pos=r[1], n_tok=r[2], need_logits=r[3],
                                              is_decode=r[4], reserved=0, req_id=r[5]) for r in rows])
        tokens = []
        for r in rows:
            for j in range(r[2]):
                pos = r[1] + j
                if r[4]:
                    tokens.append(BOS if pos == 0 else self.last_tok[(mb, r[0])])
                else:
                    tokens.append(self.lr.lib.lr_prompt_token(r[5], pos))
        tok = np.array(tokens, dtype=np.int32)
        out = {}
        # ---- GPU
        gin = None
        if not self.first:
            a16 = act_in.astype(np.float32).view(np.uint32) >> 16
            a16 = a16.astype(np.uint16)
            nat.check(nat.lib.ds_dbg_copy(self.d_act, a16.ctypes.data, a16.nbytes))
            gin = self.d_act
        if self.first and self.last:
            # ids of the previous circuit loop back inside the stage
            gin = None
        elif self.first and ids_in is not None and len(ids_in):
            ii = np.ascontiguousarray(ids_in, dtype=np.int32)
            nat.check(nat.lib.ds_dbg_copy(self.d_ids, ii.ctypes.data, ii.nbytes))
            gin = self.d_ids
        gout = self.d_ids if self.last else None
        nat.check(nat.lib.ds_stage_step(self.st, mb, arr, len(rows), gin, gout))
        nat.check(nat.lib.ds_stage_sync(self.st))
        if self.last:
            ids = np.zeros(R, dtype=np.int32)
            if R:
                nat.check(nat.lib.ds_dbg_copy(ids.ctypes.data, self.d_ids, R * 4))
            lg = np.zeros((R, V), dtype=np.float32)
            n = C.c_int64(0)
            if R:
                nat.check(nat.lib.ds_stage_logits(self.st, lg.ctypes.data, lg.size, C.byref(n)))
            out["gpu_ids"], out["gpu_logits"] = ids, lg
            # next decode input per slot = what the GPU sampled
            k = 0
            for r in rows:
                if r[3]:
                    self.last_tok[(mb, r[0])] = int(ids[k])
                    k += 1
        else:
            ptr, nbytes, nout = C.c_void_p(), C.c_int64(), C.c_int64()
            nat.check(nat.lib.ds_stage_output(self.st, C.byref(ptr), C.byref(nbytes), C.byref(nout)))
            h = np.zeros((T, d), dtype=np.uint16)
            nat.check(nat.lib.ds_dbg_copy(h.ctypes.data, ptr, h.nbytes))
            out["gpu_act"] = (h.astype(np.uint32) << 16).view(np.float32)
        # ---- CPU oracle
        lr_rows = (nat.Row * len(rows))(*arr)
        cin = None if self.first else np.ascontiguousarray(act_in, dtype=np.float32)
        cact = np.zeros((T, d), dtype=np.float32)
        clog = np.zeros((max(R, 1), V), dtype=np.float32)
        cids = np.zeros(max(R, 1), dtype=np.int32)
        rc = self.lr.lib.lr_stage_step(self.cs, mb, self.max_slots, lr_rows, len(rows),
                                       tok.ctypes.data, None if cin is None else cin.ctypes.data,
                                       cact.ctypes.data, clog.ctypes.data if self.last else None,
                                       cids.ctypes.data)
        assert rc == 0
        out["cpu_act"] = cact
        if self.last:
            out["cpu_logits"], out["cpu_ids"] = clog[:R], cids[:R]
        return out


def logits_ok(gpu, cpu, atol=0.08, rtol=0.02):
    err = np.abs(gpu - cpu)
    return bool(np.all(err <= atol + rtol * np.abs(cpu))), float(err.max())


def deep_logits_ok(gpu, cpu):
    """Whole-model / multi-layer-stage tolerance: bf16 rounding differences
    compound with depth (measured at 32 layers: RMS |dlogit| 0.021 at logit RMS 1.0, max 0.113 over
    128256 logits). Per row RMS(d) <= 0.04 RMS(logits) and every |d| <= 0.16 + 0.02 |logit|; a
    real defect (a wrong head, position or page) moves the RMS error to O(RMS(logits))."""
    err = np.abs(gpu - cpu)
    rms_rel = np.sqrt((err ** 2).mean(axis=1)) / np.sqrt((cpu ** 2).mean(axis=1))
    ok = bool(np.all(rms_rel <= 0.04) and np.all(err <= 0.16 + 0.02 * np.abs(cpu)))
    return ok, float(rms_rel.max()), float(err.max())


def deep_act_ok(gpu, cpu):
    """Activations after a multi-layer stage: per row RMS(d) <= 0.02 RMS(x) and max |d| <= 0.06
    of the row's max |x| (measured at 10 layers of 70B: max 0.033)."""
    err = np.abs(gpu - cpu)
    rms_rel = np.sqrt((err ** 2).mean(axis=1)) / np.maximum(np.sqrt((cpu ** 2).mean(axis=1)), 1e-30)
    max_rel = err.max(axis=1) / np.maximum(np.abs(cpu).max(axis=1), 1e-30)
    return bool(np.all(rms_rel <= 0.02) and np.all(max_rel <= 0.06)), float(rms_rel.max()), float(max_rel.max())


def greedy_ok(gpu_ids, cpu_logits, margin):
    """GPU argmax must equal the oracle's wherever the oracle's top-2 margin exceeds `margin`."""
    bad = []
    for i, row in enumerate(cpu_logits):
        top = np.argsort(row)[-2:]
        m = row[top[1]] - row[top[0]]
        if m > margin and int(gpu_ids[i]) != int(np.argmax(row)):
            bad.append((i, int(gpu_ids[i]), int(np.argmax(row)), float(m)))
    return bad


def random_act(T, d, seed):
    rng = np.random.default_rng(seed)
    return round_bf16(rng.standard_normal((T, d)).astype(np.float32))
