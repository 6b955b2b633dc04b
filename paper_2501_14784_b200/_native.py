"""ctypes binding of libdeserve_b200.so (C ABI: include/deserve.h).

The library is built in-tree (``make -C paper_2501_14784_b200/csrc``) and is the only
implementation of the stage-step path: there is no Python or CPU fallback. If the shared object
is missing, importing this module raises.
"""
from __future__ import annotations

import ctypes as C
import os

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_HERE, "libdeserve_b200.so")

DS_OK, DS_ERR_ARG, DS_ERR_PLAN, DS_ERR_RUNTIME, DS_ERR_NO_DEVICE = 0, 1, 2, 3, 4


class DsError(RuntimeError):
    """A non-zero ds_status; ``code`` mirrors the reference error classes (cli.cpp:219-231)."""

    def __init__(self, code: int, msg: str):
        super().__init__(f"ds_status {code}: {msg}")
        self.code = code


class ConfigError(DsError):
    pass


class PlanError(DsError):
    pass


class SimError(DsError):
    pass


class NoDeviceError(DsError):
    pass


_ERR = {DS_ERR_ARG: ConfigError, DS_ERR_PLAN: PlanError, DS_ERR_RUNTIME: SimError,
        DS_ERR_NO_DEVICE: NoDeviceError}


class ModelDesc(C.Structure):
    _fields_ = [("n_layers", C.c_int32), ("d_model", C.c_int32), ("n_heads", C.c_int32),
                ("n_kv_heads", C.c_int32), ("d_head", C.c_int32), ("ffn", C.c_int32),
                ("vocab", C.c_int32), ("max_seq_len", C.c_int32), ("rope_theta", C.c_float),
                ("norm_eps", C.c_float)]


class Row(C.Structure):
    _fields_ = [("slot", C.c_int32), ("pos", C.c_int32), ("n_tok", C.c_int32),
                ("need_logits", C.c_int32), ("is_decode", C.c_int32), ("reserved", C.c_int32),
                ("req_id", C.c_int64)]


class GpuOpts(C.Structure):
    _fields_ = [("device0", C.c_int32), ("n_devices", C.c_int32), ("real_delay", C.c_int32),
                ("collect_tokens", C.c_int32), ("max_circuits", C.c_int64),
                ("weight_seed", C.c_uint64), ("trace", C.c_int32), ("reserved", C.c_int32)]


def _load() -> C.CDLL:
    if not os.path.exists(LIB_PATH):
        raise ImportError(f"{LIB_PATH} is not built; run `make -C {_HERE}/csrc` "
                          "(the CUDA path has no fallback)")
    lib = C.CDLL(LIB_PATH)
    I64, I32, P, S = C.c_int64, C.c_int32, C.c_void_p, C.c_char_p
    sig = {
        "ds_last_error": (S, []),
        "ds_version": (S, []),
        "ds_prompt_token_id": (I32, [I64, I32]),
        "ds_stage_time_us": (I32, [P, P, I64, I64, I64, I64, P]),
        "ds_page_bytes": (I32, [I64, I64, I64, P]),
        "ds_global_pool_size": (I32, [I64, I64, I64, P]),
        "ds_memory_budget": (I32, [I64, I64, I64, I64, I32, P]),
        "ds_request_lengths": (I32, [C.c_uint64, I64, I64, I64, I64, I64, P]),
        "ds_steady_state_throughput": (I32, [S, P]),
        "ds_plan_config": (I32, [S, S, S, I64, I64, P, C.c_size_t, P]),
        "ds_sim_config": (I32, [S, S, S, I64, I64, S, P, C.c_size_t]),
        "ds_sim_plan": (I32, [S, S, S, S, P, C.c_size_t]),
        "ds_stage_create": (I32, [I32, P, I64, I64, I32, I32, C.c_uint64, I32, I32, P]),
        "ds_stage_destroy": (I32, [P]),
        "ds_kv_create": (I32, [P, I64, I64, I64, I64, I64]),
        "ds_kv_release": (I32, [P, I32, I32]),
        "ds_kv_usage": (I32, [P, I32, P, P]),
        "ds_swap_in": (I32, [P, I32, I32, I64, P, P]),
        "ds_stage_step": (I32, [P, I32, P, I64, P, P]),
        "ds_stage_output": (I32, [P, P, P, P]),
        "ds_stage_sync": (I32, [P]),
        "ds_stage_stream": (I32, [P, P]),
        "ds_stage_logits": (I32, [P, P, I64, P]),
        "ds_kv_resident": (I32, [P, I32, P]),
        "ds_kv_ready": (I32, [P, I32, P, I64, P]),
        "ds_kv_reset": (I32, [P]),
        "ds_session_create": (I32, [S, S, S, I64, I64, P, P, P]),
        "ds_session_run": (I32, [P, I32, I32, P, C.c_size_t, P]),
        "ds_session_destroy": (I32, [P]),
        "ds_nccl_unique_id": (I32, [P]),
        "ds_session_create_rank": (I32, [S, S, S, I64, I64, P, P, I32, I32, P, P]),
        "ds_stage_profile": (I32, [P, I32]),
        "ds_stage_kernel_stats": (I32, [P, P, C.c_size_t, P]),
        "ds_schedule_config": (I32, [S, S, S, I64, I64, I64, P, C.c_size_t, P]),
        "ds_gpu_run_config": (I32, [S, S, S, I64, I64, P, P, P, C.c_size_t, P]),
        "ds_stage_step_events": (I32, [P, P, P, P]),
        "ds_swap_stats": (I32, [P, P]),
        "ds_swap_events": (I32, [P, P, P, P, P]),
        "ds_stage_logits_device": (I32, [P, P, P]),
        "ds_session_trace": (I32, [P, S, I64, I32, I64, I64, P, C.c_size_t, P]),
        "ds_trace_merge": (I32, [P, I32, S]),
        "ds_trace_report": (I32, [S, I64, I64, I64, C.c_uint64, P, C.c_size_t]),
        "ds_run": (I32, [S, S, S, I64, I64, P, P, S, P, C.c_size_t, P]),
        "ds_session_capture": (I32, [P, P, I64]),
        "ds_session_limit": (I32, [P, I64, P]),
        "ds_report_kv": (I32, [S, S, I64, S, P, C.c_size_t, P]),
        "ds_report_kv_priced": (I32, [S, S, I64, S, S, P, C.c_size_t, P]),
        "ds_sweep_csv": (I32, [P, I32, S, P, P, C.c_size_t, P]),
        "ds_session_captured": (I32, [P, P, P, I64, P]),
        "ds_dbg_gemm": (I32, [P, P, I32, I32, I32, I32, P, I32, P]),
        "ds_dbg_gemm_norm": (I32, [P, P, I32, I32, I32, P, P, I32, C.c_float, P, P, P]),
        "ds_dbg_has_device": (I32, [P]),
        "ds_dbg_gemm_bench": (I32, [I32, I32, I32, I32, I32, I32, P]),
        "ds_dbg_gemm_plan": (I32, [I32, I32, I32, P]),
        "ds_dbg_alloc": (I32, [I32, I64, P]),
        "ds_dbg_free": (I32, [P]),
        "ds_dbg_copy": (I32, [P, P, I64]),
    }
    for name, (res, args) in sig.items():
        fn = getattr(lib, name)
        fn.restype = res
        fn.argtypes = args
    return lib


lib = _load()


def check(status: int) -> None:
    if status != DS_OK:
        msg = lib.ds_last_error().decode(errors="replace")
        raise _ERR.get(status, DsError)(status, msg)


def n_devices() -> int:
    n = C.c_int32(0)
    check(lib.ds_dbg_has_device(C.byref(n)))
    return n.value


def exported_symbols() -> list[str]:
    """Every ds_* entry point declared in include/deserve.h."""
    import re
    hdr = os.path.join(os.path.dirname(_HERE), "include", "deserve.h")
    return sorted(set(re.findall(r"\b(ds_[a-z0-9_]+)\s*\(", open(hdr).read())))
