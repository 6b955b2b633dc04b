"""TEST INFRASTRUCTURE ONLY — parity checkers. Imported by tests/, __graft_entry__.smoke() and
bench.py's cpu_baseline / --impl reference legs, never by the product package.

* ``Ref``  — the UNMODIFIED reference pipesim library (oracle/_ref/libpipesim_ref.so, compiled
  from /root/reference/proj/src by oracle/Makefile) behind a small C shim (ref_shim.cpp).
* ``LlamaRef`` — the CPU restatement of the stage forward (oracle/llama_ref.c); the reference has
  no arithmetic for this part, so it is pinned only by its own conventions.
"""
from __future__ import annotations

import ctypes as C
import json
import os

HERE = os.path.dirname(os.path.abspath(__file__))
# model dims and the weight seed of the workloads (restated here so the checkers and the CPU
# baselines never import the product package; must equal paper_2501_14784_b200.pipeline's)
MODEL_DIMS = {
    "tiny-llama": dict(n_layers=4, d_model=256, n_heads=4, n_kv_heads=2, d_head=64, ffn=768,
                       vocab=128256, max_seq_len=8192, rope_theta=500000.0, norm_eps=1e-5),
    "llama3-8b": dict(n_layers=32, d_model=4096, n_heads=32, n_kv_heads=8, d_head=128, ffn=14336,
                      vocab=128256, max_seq_len=8192, rope_theta=500000.0, norm_eps=1e-5),
    "llama3-70b-bf16": dict(n_layers=80, d_model=8192, n_heads=64, n_kv_heads=8, d_head=128,
                            ffn=28672, vocab=128256, max_seq_len=8192, rope_theta=500000.0,
                            norm_eps=1e-5),
}
WEIGHT_SEED = 0x5EED0001
REF_SO = os.path.join(HERE, "_ref", "libpipesim_ref.so")
LLAMA_SO = os.path.join(HERE, "_build", "libllama_ref.so")


def _b(s):
    return None if s is None else (s.encode() if isinstance(s, str) else s)


class RefError(RuntimeError):
    pass


class Ref:
    """Compiled reference (pipesim) through ref_shim.cpp."""

    def __init__(self):
        if not os.path.exists(REF_SO):
            raise FileNotFoundError(f"{REF_SO} missing: run `make -C {HERE}`")
        lib = C.CDLL(REF_SO)
        L, S, P = C.c_longlong, C.c_char_p, C.c_void_p
        lib.ref_last_error.restype = S
        for name, args in {
            "ref_plan_config": [S, S, S, L, L, P, C.c_size_t],
            "ref_sim_config": [S, S, S, L, L, S, P, C.c_size_t],
            "ref_sim_plan": [S, S, S, S, P, C.c_size_t],
            "ref_stage_time": [P, P, L, L, L, L, P],
            "ref_page_bytes": [L, L, L, P],
            "ref_global_pool_size": [L, L, L, P],
            "ref_memory_budget": [L, L, L, L, C.c_int, P],
            "ref_replay_check": [S, S, P, C.c_size_t],
            "ref_windowed_stats": [S, L, L, C.c_int, P],
            "ref_request": [C.c_ulonglong, L, L, L, L, L, P],
            "ref_report_kv": [S, S, S, L, L, P, C.c_size_t],
            "ref_report_kv_priced": [S, S, S, L, L, P, C.c_size_t],
            "ref_sweep_csv": [S, S, P, C.c_size_t],
        }.items():
            getattr(lib, name).argtypes = args
            getattr(lib, name).restype = C.c_int
        lib.ref_steady_state.argtypes = [S]
        lib.ref_steady_state.restype = C.c_double
        self.lib = lib

    def _ok(self, rc):
        if rc != 0:
            raise RefError(self.lib.ref_last_error().decode())

    def plan_config(self, text, cdir="", policy=None, latency_us=-1, nb=-1) -> str:
        buf = C.create_string_buffer(1 << 20)
        self._ok(self.lib.ref_plan_config(_b(text), _b(cdir), _b(policy or ""), latency_us, nb,
                                          buf, len(buf)))
        return buf.value.decode()

    def sim_config(self, text, cdir="", policy=None, latency_us=-1, nb=-1, trace_path=None) -> dict:
        buf = C.create_string_buffer(1 << 16)
        self._ok(self.lib.ref_sim_config(_b(text), _b(cdir), _b(policy or ""), latency_us, nb,
                                         _b(trace_path or ""), buf, len(buf)))
        return json.loads(buf.value.decode())

    def sim_plan(self, text, plan_json, cdir="", trace_path=None) -> dict:
        buf = C.create_string_buffer(1 << 16)
        self._ok(self.lib.ref_sim_plan(_b(text), _b(cdir), _b(plan_json), _b(trace_path or ""),
                                       buf, len(buf)))
        return json.loads(buf.value.decode())

    def report_kv(self, text, cdir="", policy=None, latency_us=-1, nb=-1) -> str:
        buf = C.create_string_buffer(1 << 16)
        self._ok(self.lib.ref_report_kv(_b(text), _b(cdir), _b(policy or ""), latency_us, nb, buf,
                                        len(buf)))
        return buf.value.decode()

    def report_kv_priced(self, text, cdir="", policy=None, latency_us=-1, nb=-1) -> str:
        buf = C.create_string_buffer(1 << 16)
        self._ok(self.lib.ref_report_kv_priced(_b(text), _b(cdir), _b(policy or ""), latency_us, nb,
                                               buf, len(buf)))
        return buf.value.decode()

    def sweep_csv(self, text, cdir="") -> str:
        buf = C.create_string_buffer(1 << 16)
        self._ok(self.lib.ref_sweep_csv(_b(text), _b(cdir), buf, len(buf)))
        return buf.value.decode()

    def stage_time(self, table, batch, layers, ref_layers) -> int:
        b = (C.c_longlong * len(table))(*[x[0] for x in table])
        t = (C.c_longlong * len(table))(*[x[1] for x in table])
        out = C.c_longlong(0)
        self._ok(self.lib.ref_stage_time(b, t, len(table), batch, layers, ref_layers, C.byref(out)))
        return out.value

    def page_bytes(self, kvpt, layers, total) -> int:
        out = C.c_longlong(0)
        self._ok(self.lib.ref_page_bytes(kvpt, layers, total, C.byref(out)))
        return out.value

    def global_pool_size(self, w, t, page) -> int:
        out = C.c_longlong(0)
        self._ok(self.lib.ref_global_pool_size(w, t, page, C.byref(out)))
        return out.value

    def memory_budget(self, mem, weights, nb, mg, offload) -> list[int]:
        out = (C.c_longlong * 5)()
        self._ok(self.lib.ref_memory_budget(mem, weights, nb, mg, int(offload), out))
        return list(out)

    def replay_check(self, trace_path, plan_json) -> list[str]:
        buf = C.create_string_buffer(1 << 20)
        self._ok(self.lib.ref_replay_check(_b(trace_path), _b(plan_json), buf, len(buf)))
        return [x for x in buf.value.decode().splitlines() if x]

    def windowed_stats(self, trace_path, start, end, completed=False):
        out = (C.c_longlong * 3)()
        self._ok(self.lib.ref_windowed_stats(_b(trace_path), start, end, int(completed), out))
        return tuple(out)

    def steady_state(self, plan_json) -> float:
        return self.lib.ref_steady_state(_b(plan_json))

    def request(self, seed, pmin, pmax, omin, omax, index):
        out = (C.c_longlong * 2)()
        self._ok(self.lib.ref_request(seed, pmin, pmax, omin, omax, index, out))
        return out[0], out[1]


BINDING_SO = os.path.join(HERE, "_ref", "libb200_binding.so")


def binding_run_and_check(config_text: str, config_dir: str, plan_json: str, model_desc, gpu_opts,
                          trace_path: str) -> dict:
    """integration/run_on_b200.cpp -- the reference-side binding compiled against the reference
    headers -- runs the config on the GPU (ds_run) into a pipesim::SimResult and applies the
    reference's replay_check / windowed_stats to it in C++. Raises RefError with the binding's
    message (e.g. the product's "no CUDA device" on a CPU box)."""
    lib = C.CDLL(BINDING_SO)
    lib.b200_run_and_check.argtypes = [C.c_char_p] * 3 + [C.c_void_p] * 2 + [C.c_char_p, C.c_void_p,
                                                                           C.c_size_t]
    lib.b200_run_and_check.restype = C.c_int
    buf = C.create_string_buffer(1 << 16)
    rc = lib.b200_run_and_check(_b(config_text), _b(config_dir), _b(plan_json), C.byref(model_desc),
                                C.byref(gpu_opts), _b(trace_path), buf, len(buf))
    if rc != 0:
        raise RefError(buf.value.decode())
    return json.loads(buf.value.decode())


class LrModel(C.Structure):
    _fields_ = [("n_layers", C.c_int32), ("d_model", C.c_int32), ("n_heads", C.c_int32),
                ("n_kv_heads", C.c_int32), ("d_head", C.c_int32), ("ffn", C.c_int32),
                ("vocab", C.c_int32), ("max_seq_len", C.c_int32), ("rope_theta", C.c_float),
                ("norm_eps", C.c_float)]


class LlamaRef:
    """CPU oracle of one stage (oracle/llama_ref.c), multithreaded with OpenMP."""

    def __init__(self):
        if not os.path.exists(LLAMA_SO):
            raise FileNotFoundError(f"{LLAMA_SO} missing: run `make -C {HERE} llama`")
        lib = C.CDLL(LLAMA_SO)
        P = C.c_void_p
        lib.lr_weight.argtypes = [C.c_uint64, C.c_uint64, C.c_int64, C.c_float]
        lib.lr_weight.restype = C.c_float
        lib.lr_prompt_token.argtypes = [C.c_int64, C.c_int32]
        lib.lr_prompt_token.restype = C.c_int32
        lib.lr_stage_create.argtypes = [P, C.c_int32, C.c_int32, C.c_int32, C.c_int32, C.c_uint64,
                                        C.c_int32]
        lib.lr_stage_create.restype = P
        lib.lr_stage_destroy.argtypes = [P]
        lib.lr_stage_step.argtypes = [P, C.c_int32, C.c_int32, P, C.c_int32, P, P, P, P, P]
        lib.lr_stage_step.restype = C.c_int
        self.lib = lib


def replay_circuits(schedule: dict, plan: dict, dims: dict, seed: int, gpu_tokens):
    """Runs the schedule's circuits through the CPU oracle stages (all stages of the plan, in
    circuit order), teacher-forcing decode inputs with the GPU's sampled ids. Returns, per
    circuit, the oracle logits of the rows that sample a token."""
    import numpy as np
    lr = LlamaRef()
    m = LrModel(**dims)
    S = len(plan["stages"])
    B = plan["stages"][0]["batch_size_per_microbatch"]
    NB = plan["n_microbatches"]
    stages = [lr.lib.lr_stage_create(C.byref(m), s["layer_begin"], s["layer_end"], int(i == 0),
                                     int(i == S - 1), seed, NB * B)
              for i, s in enumerate(plan["stages"])]

    class Row(C.Structure):
        _fields_ = [("slot", C.c_int32), ("pos", C.c_int32), ("n_tok", C.c_int32),
                    ("need_logits", C.c_int32), ("is_decode", C.c_int32), ("reserved", C.c_int32),
                    ("req_id", C.c_int64)]
    last, out = {}, []
    try:
        for ci, c in enumerate(schedule["circuits"]):
            rows = c["rows"]
            arr = (Row * len(rows))(*[Row(r[0], r[1], r[2], r[3], r[4], 0, r[5]) for r in rows])
            toks = []
            for r in rows:
                for j in range(r[2]):
                    pos = r[1] + j
                    toks.append((128000 if pos == 0 else last[(c["mb"], r[0])]) if r[4]
                                else lr.lib.lr_prompt_token(r[5], pos))
            T = sum(r[2] for r in rows)
            R = sum(r[3] for r in rows)
            tok = np.array(toks, dtype=np.int32)
            a = np.zeros((T, dims["d_model"]), dtype=np.float32)
            b = np.zeros_like(a)
            lg = np.zeros((max(R, 1), dims["vocab"]), dtype=np.float32)
            ids = np.zeros(max(R, 1), dtype=np.int32)
            for i in range(S):
                src, dst = (a, b) if i % 2 == 0 else (b, a)
                rc = lr.lib.lr_stage_step(stages[i], c["mb"], B, arr, len(rows), tok.ctypes.data,
                                          src.ctypes.data if i else None, dst.ctypes.data,
                                          lg.ctypes.data if i == S - 1 else None, ids.ctypes.data)
                if rc != 0:
                    raise RefError("oracle stage step failed")
            k = 0
            for r in rows:
                if r[3]:
                    last[(c["mb"], r[0])] = gpu_tokens[ci][k]
                    k += 1
            out.append(lg[:R].copy())
    finally:
        for s in stages:
            lr.lib.lr_stage_destroy(s)
    return out


class LrRow(C.Structure):
    """Row descriptor of llama_ref.h (same layout as the product's ds_row; defined here so the
    checkers never import the product package)."""
    _fields_ = [("slot", C.c_int32), ("pos", C.c_int32), ("n_tok", C.c_int32),
                ("need_logits", C.c_int32), ("is_decode", C.c_int32), ("reserved", C.c_int32),
                ("req_id", C.c_int64)]


def replay_requests(schedule: dict, dims: dict, seed: int, reqs, gpu_tokens):
    """Whole-model oracle (all layers, embedding and LM head in one CPU stage) over the rows of
    the selected requests only, in the schedule's circuit order: requests are independent (a row
    attends only to its own request's KV), so the logits of their sampled rows equal those of the
    full circuits. Decode inputs are teacher-forced with the GPU's sampled ids (gpu_tokens: per
    circuit, the ids of its need_logits rows in row order). Returns (meta [n, 3] = circuit,
    req_id, position; logits [n, vocab]) in execution order (the order ds_session_captured uses)."""
    import numpy as np
    lr = LlamaRef()
    m = LrModel(**dims)
    sel = {q: i for i, q in enumerate(sorted(reqs))}
    st = lr.lib.lr_stage_create(C.byref(m), 0, dims["n_layers"], 1, 1, seed, len(sel))
    last, meta, out = {}, [], []
    try:
        for ci, c in enumerate(schedule["circuits"]):
            rows, toks, k = [], [], 0
            for r in c["rows"]:
                if r[5] in sel:
                    rows.append(r)
                    for j in range(r[2]):
                        pos = r[1] + j
                        toks.append((128000 if pos == 0 else last[r[5]]) if r[4]
                                    else lr.lib.lr_prompt_token(r[5], pos))
            for r in c["rows"]:  # teacher forcing: the GPU's sample of each selected row
                if r[3]:
                    if r[5] in sel:
                        last[r[5]] = int(gpu_tokens[ci][k])
                    k += 1
            if not rows:
                continue
            arr = (LrRow * len(rows))(*[LrRow(sel[r[5]], r[1], r[2], r[3], r[4], 0, r[5])
                                        for r in rows])
            T = sum(r[2] for r in rows)
            R = sum(r[3] for r in rows)
            tok = np.array(toks, dtype=np.int32)
            act = np.zeros((T, dims["d_model"]), dtype=np.float32)
            lg = np.zeros((max(R, 1), dims["vocab"]), dtype=np.float32)
            ids = np.zeros(max(R, 1), dtype=np.int32)
            if lr.lib.lr_stage_step(st, 0, len(sel), arr, len(rows), tok.ctypes.data, None,
                                    act.ctypes.data, lg.ctypes.data, ids.ctypes.data) != 0:
                raise RefError("oracle stage step failed")
            i = 0
            for r in rows:
                if r[3]:
                    meta.append((ci, r[5], r[1] + r[2] - 1))
                    out.append(lg[i].copy())
                    i += 1
    finally:
        lr.lib.lr_stage_destroy(st)
    return np.array(meta, dtype=np.int64).reshape(-1, 3), np.array(out, dtype=np.float32)


class CircuitTimer:
    """Times the CPU stage forward (oracle/llama_ref.c, OpenMP on every host core) on whole
    circuits of a single-stage schedule: all layers + embedding + LM head, the circuit's exact
    rows (prompt chunks and decode rows at their positions). Only time is measured: each timed
    circuit starts from zeroed KV (decode rows still attend over all their positions), so any
    circuit of the schedule can be timed without replaying its history."""

    def __init__(self, dims: dict, seed: int, max_slots: int):
        self.lr = LlamaRef()
        self.lr.lib.lr_stage_reset_kv.argtypes = [C.c_void_p]
        self.dims = dims
        self.max_slots = max_slots
        m = LrModel(**dims)
        self.st = self.lr.lib.lr_stage_create(C.byref(m), 0, dims["n_layers"], 1, 1, seed, max_slots)

    def close(self):
        if self.st:
            self.lr.lib.lr_stage_destroy(self.st)
            self.st = None

    def time(self, circuit: dict) -> float:
        import time

        import numpy as np
        rows = circuit["rows"]
        arr = (LrRow * len(rows))(*[LrRow(r[0], r[1], r[2], r[3], r[4], 0, r[5]) for r in rows])
        toks = []
        for r in rows:
            for j in range(r[2]):
                pos = r[1] + j
                toks.append((128000 if pos == 0 else 1000) if r[4] else self.lr.lib.lr_prompt_token(r[5], pos))
        T = len(toks)
        R = sum(r[3] for r in rows)
        tok = np.array(toks, dtype=np.int32)
        act = np.zeros((T, self.dims["d_model"]), dtype=np.float32)
        lg = np.zeros((max(R, 1), self.dims["vocab"]), dtype=np.float32)
        ids = np.zeros(max(R, 1), dtype=np.int32)
        self.lr.lib.lr_stage_reset_kv(self.st)
        t0 = time.perf_counter()
        rc = self.lr.lib.lr_stage_step(self.st, 0, self.max_slots, arr, len(rows), tok.ctypes.data,
                                       None, act.ctypes.data, lg.ctypes.data, ids.ctypes.data)
        dt = time.perf_counter() - t0
        if rc != 0:
            raise RefError("oracle stage step failed")
        return dt


def load_schedule_fixture(path: str) -> list:
    import gzip
    with gzip.open(path, "rt") as f:
        return json.load(f)


def greedy_mismatches(oracle_logits, gpu_tokens, margin):
    """(checked, mismatched): rows whose oracle top-2 margin exceeds `margin` must agree."""
    import numpy as np
    checked = bad = 0
    for ci, lg in enumerate(oracle_logits):
        for k, row in enumerate(lg):
            top = np.sort(row)[-2:]
            if top[1] - top[0] > margin:
                checked += 1
                bad += int(int(np.argmax(row)) != int(gpu_tokens[ci][k]))
    return checked, bad
