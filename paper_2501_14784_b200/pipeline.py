"""Python mirror of the reference's plan/run interface over the C ABI.

Reference names and meaning:
  plan_config  -> pipesim::plan (src/planner.cpp:140-276) on a config document
  sim_config   -> pipesim::run  (src/sim.cpp:591-595), virtual clock, executor = ours
  sim_plan     -> run() on an explicit PipelinePlan JSON
Errors raise ConfigError / PlanError / SimError like the reference's exception classes.
"""
from __future__ import annotations

import ctypes as C
import json
import os

from ._native import check, lib


def _b(s):
    return None if s is None else (s.encode() if isinstance(s, str) else s)


def read_config(path: str) -> tuple[str, str]:
    return open(path).read(), os.path.dirname(os.path.abspath(path))


def plan_config(config_text: str, config_dir: str = "", policy: str | None = None,
                latency_us: int = -1, nb_override: int = -1) -> str:
    need = C.c_size_t(0)
    check(lib.ds_plan_config(_b(config_text), _b(config_dir), _b(policy or ""), latency_us,
                             nb_override, None, 0, C.byref(need)))
    buf = C.create_string_buffer(need.value)
    check(lib.ds_plan_config(_b(config_text), _b(config_dir), _b(policy or ""), latency_us,
                             nb_override, buf, need.value, None))
    return buf.value.decode()


def sim_config(config_text: str, config_dir: str = "", policy: str | None = None,
               latency_us: int = -1, nb_override: int = -1, trace_path: str | None = None) -> dict:
    buf = C.create_string_buffer(1 << 16)
    check(lib.ds_sim_config(_b(config_text), _b(config_dir), _b(policy or ""), latency_us,
                            nb_override, _b(trace_path or ""), buf, len(buf)))
    return json.loads(buf.value.decode())


def sim_plan(config_text: str, plan_json: str, config_dir: str = "",
             trace_path: str | None = None) -> dict:
    buf = C.create_string_buffer(1 << 16)
    check(lib.ds_sim_plan(_b(config_text), _b(config_dir), _b(plan_json), _b(trace_path or ""),
                          buf, len(buf)))
    return json.loads(buf.value.decode())


def stage_time_us(table: list[tuple[int, int]], batch: int, layers: int, ref_layers: int) -> int:
    b = (C.c_int64 * len(table))(*[x[0] for x in table])
    t = (C.c_int64 * len(table))(*[x[1] for x in table])
    out = C.c_int64(0)
    check(lib.ds_stage_time_us(b, t, len(table), batch, layers, ref_layers, C.byref(out)))
    return out.value


def page_bytes(kv_bytes_per_token: int, layers: int, total_layers: int) -> int:
    out = C.c_int64(0)
    check(lib.ds_page_bytes(kv_bytes_per_token, layers, total_layers, C.byref(out)))
    return out.value


def global_pool_size(pcie: int, stage_time: int, page: int) -> int:
    out = C.c_int64(0)
    check(lib.ds_global_pool_size(pcie, stage_time, page, C.byref(out)))
    return out.value


def memory_budget(mem: int, weights: int, n_mb: int, m_global: int, offload: bool) -> list[int]:
    out = (C.c_int64 * 5)()
    check(lib.ds_memory_budget(mem, weights, n_mb, m_global, int(offload), out))
    return list(out)


def request_lengths(seed: int, pmin: int, pmax: int, omin: int, omax: int, index: int):
    out = (C.c_int64 * 2)()
    check(lib.ds_request_lengths(seed, pmin, pmax, omin, omax, index, out))
    return out[0], out[1]


def steady_state_throughput(plan_json: str) -> float:
    out = C.c_double(0)
    check(lib.ds_steady_state_throughput(_b(plan_json), C.byref(out)))
    return out.value


# --------------------------------------------------------------------------- GPU path ----
# Architecture dims per config model name (the reference ModelSpec carries only byte totals;
# kv_bytes_per_token must equal 4 * n_kv * d_head * n_layers, checked by the executor).
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


def model_desc(name_or_dims):
    from ._native import ModelDesc
    d = MODEL_DIMS[name_or_dims] if isinstance(name_or_dims, str) else name_or_dims
    return ModelDesc(**d)


def schedule_config(config_text: str, config_dir: str = "", policy=None, latency_us=-1,
                    nb_override=-1, max_circuits=0) -> dict:
    need = C.c_size_t(0)
    check(lib.ds_schedule_config(_b(config_text), _b(config_dir), _b(policy or ""), latency_us,
                                 nb_override, max_circuits, None, 0, C.byref(need)))
    buf = C.create_string_buffer(need.value)
    check(lib.ds_schedule_config(_b(config_text), _b(config_dir), _b(policy or ""), latency_us,
                                 nb_override, max_circuits, buf, need.value, None))
    return json.loads(buf.value.decode())


def gpu_run_config(config_text: str, config_dir: str = "", policy=None, latency_us=-1,
                   nb_override=-1, model=None, device0=0, n_devices=0, real_delay=True,
                   collect_tokens=False, max_circuits=0, weight_seed=WEIGHT_SEED) -> dict:
    """Plan + schedule + execute on GPUs (replay mode). Raises on any CUDA/KV/runtime error."""
    from ._native import GpuOpts
    if model is None:
        model = json.loads(config_text)["model"]["name"]
    md = model_desc(model)
    opts = GpuOpts(device0=device0, n_devices=n_devices, real_delay=int(real_delay),
                   collect_tokens=int(collect_tokens), max_circuits=max_circuits,
                   weight_seed=weight_seed)
    need = C.c_size_t(0)
    cap = 1 << 26
    buf = C.create_string_buffer(cap)
    st = lib.ds_gpu_run_config(_b(config_text), _b(config_dir), _b(policy or ""), latency_us,
                               nb_override, C.byref(md), C.byref(opts), buf, cap, C.byref(need))
    check(st)
    return json.loads(buf.value.decode())


def run(config_text: str, config_dir: str = "", policy=None, latency_us=-1, nb_override=-1,
        model=None, device0=0, n_devices=0, real_delay=True, collect_tokens=False,
        max_circuits=0, weight_seed=WEIGHT_SEED, trace_path: str | None = None) -> dict:
    """The reference's run() with real stage forwards (ds_run): returns
    {"report": SimReport fields of the hardware run, "gpu": executor report}; the real-clock
    EventTrace goes to trace_path."""
    from ._native import GpuOpts
    if model is None:
        model = json.loads(config_text)["model"]["name"]
    md = model_desc(model)
    opts = GpuOpts(device0=device0, n_devices=n_devices, real_delay=int(real_delay),
                   collect_tokens=int(collect_tokens), max_circuits=max_circuits,
                   weight_seed=weight_seed, trace=1)
    cap = 1 << 26
    buf = C.create_string_buffer(cap)
    need = C.c_size_t(0)
    check(lib.ds_run(_b(config_text), _b(config_dir), _b(policy or ""), latency_us, nb_override,
                     C.byref(md), C.byref(opts), _b(trace_path or ""), buf, cap, C.byref(need)))
    return json.loads(buf.value.decode())


def trace_merge(paths: list[str], out_path: str) -> None:
    arr = (C.c_char_p * len(paths))(*[_b(p) for p in paths])
    check(lib.ds_trace_merge(arr, len(paths), _b(out_path)))


def trace_report(trace_path: str, n_stages: int, w0_us: int, w1_us: int, seed: int = 0) -> dict:
    buf = C.create_string_buffer(1 << 16)
    check(lib.ds_trace_report(_b(trace_path), n_stages, w0_us, w1_us, seed, buf, len(buf)))
    return json.loads(buf.value.decode())


def report_kv(report: dict, plan_json: str, latency_us: int, policy: str, pricing=None) -> str:
    """report.kv text of a report (reference report_to_kv, sweep.cpp:146-195). `pricing` (a config
    document's "pricing" object, e.g. {"preset": "whattomine-8x4090"}) appends the profit block of
    the reference's analyze (economics.cpp:21-59), as report_to_kv does with a ProfitAnalysis."""
    need = C.c_size_t(0)
    rj = _b(json.dumps(report))
    if pricing is None:
        check(lib.ds_report_kv(rj, _b(plan_json), latency_us, _b(policy), None, 0, C.byref(need)))
        buf = C.create_string_buffer(need.value)
        check(lib.ds_report_kv(rj, _b(plan_json), latency_us, _b(policy), buf, need.value, None))
        return buf.value.decode()
    pj = _b(pricing if isinstance(pricing, str) else json.dumps(pricing))
    check(lib.ds_report_kv_priced(rj, _b(plan_json), latency_us, _b(policy), pj, None, 0,
                                  C.byref(need)))
    buf = C.create_string_buffer(need.value)
    check(lib.ds_report_kv_priced(rj, _b(plan_json), latency_us, _b(policy), pj, buf, need.value,
                                  None))
    return buf.value.decode()


def sweep_csv(latencies, policies, throughput) -> str:
    """sweep.csv text (reference SweepResult::to_csv, sweep.cpp:68-82); throughput[p][l], None =
    failed."""
    lat = (C.c_int64 * len(latencies))(*latencies)
    flat = [float("nan") if v is None else float(v) for row in throughput for v in row]
    vals = (C.c_double * len(flat))(*flat)
    need = C.c_size_t(0)
    pol = _b(",".join(policies))
    check(lib.ds_sweep_csv(lat, len(latencies), pol, vals, None, 0, C.byref(need)))
    buf = C.create_string_buffer(need.value)
    check(lib.ds_sweep_csv(lat, len(latencies), pol, vals, buf, need.value, None))
    return buf.value.decode()


class Session:
    """A planned + scheduled pipeline with its GPU stages built once (ds_session_*)."""

    def __init__(self, config_text: str, config_dir: str = "", policy=None, latency_us=-1,
                 nb_override=-1, model=None, device0=0, n_devices=0, real_delay=True,
                 max_circuits=0, weight_seed=WEIGHT_SEED, trace=False):
        from ._native import GpuOpts
        if model is None:
            model = json.loads(config_text)["model"]["name"]
        self._md = model_desc(model)
        self._opts = GpuOpts(device0=device0, n_devices=n_devices, real_delay=int(real_delay),
                             collect_tokens=0, max_circuits=max_circuits, weight_seed=weight_seed,
                             trace=int(trace))
        self._h = C.c_void_p()
        check(lib.ds_session_create(_b(config_text), _b(config_dir), _b(policy or ""), latency_us,
                                    nb_override, C.byref(self._md), C.byref(self._opts),
                                    C.byref(self._h)))

    def run(self, profile=False, collect_tokens=False) -> dict:
        cap = 1 << 26
        buf = C.create_string_buffer(cap)
        need = C.c_size_t(0)
        check(lib.ds_session_run(self._h, int(profile), int(collect_tokens), buf, cap,
                                 C.byref(need)))
        return json.loads(buf.value.decode())

    def trace(self, trace_path: str | None = None, t0_us=-1, keep_virtual_seq=False, w0_us=-1,
              w1_us=-1) -> dict:
        """Real-clock EventTrace of the last run (written to trace_path) and its SimReport."""
        need = C.c_size_t(0)
        check(lib.ds_session_trace(self._h, _b(trace_path or ""), t0_us, int(keep_virtual_seq),
                                   w0_us, w1_us, None, 0, C.byref(need)))
        buf = C.create_string_buffer(need.value + 16)
        check(lib.ds_session_trace(self._h, None, t0_us, int(keep_virtual_seq), w0_us, w1_us, buf,
                                   len(buf), None))
        return json.loads(buf.value.decode())

    def capture(self, req_ids) -> None:
        """Copy the fp32 logits of every row sampled for these requests at each run."""
        arr = (C.c_int64 * max(len(req_ids), 1))(*req_ids)
        check(lib.ds_session_capture(self._h, arr, len(req_ids)))

    def captured(self):
        """(meta [n, 4] = circuit, req_id, position, sampled-row index; logits [n, vocab])."""
        import numpy as np
        n = C.c_int64(0)
        check(lib.ds_session_captured(self._h, None, None, 0, C.byref(n)))
        meta = np.zeros((n.value, 4), dtype=np.int64)
        lg = np.zeros((n.value, self._md.vocab), dtype=np.float32)
        check(lib.ds_session_captured(self._h, meta.ctypes.data, lg.ctypes.data, n.value,
                                      C.byref(n)))
        return meta, lg

    def close(self):
        if self._h:
            lib.ds_session_destroy(self._h)
            self._h = C.c_void_p()

    def __enter__(self):
        return self

    def __exit__(self, *a):
        self.close()
