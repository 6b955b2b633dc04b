"""Per-CTA phase trace of single GEMM launches at the 8B decode shapes (run with DS_GEMM_TRACE=1:
ds_dbg_gemm_bench prints start / loads issued / MMA done / epilogue / end per CTA to stderr).
Output: profiles/r02_gemm_trace.txt."""
import ctypes as C
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2501_14784_b200._native import check, lib  # noqa: E402

SHAPES = [(180, 6144, 4096), (180, 4096, 4096), (180, 28672, 4096), (180, 4096, 14336),
          (64, 6144, 4096), (256, 4096, 4096)]

for T, N, K in SHAPES:
    ms = C.c_float(0)
    check(lib.ds_dbg_gemm_bench(T, N, K, 0, 20, 0, C.byref(ms)))
    print("T N K", T, N, K, "us", ms.value * 1e3, flush=True)
