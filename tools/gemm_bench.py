"""GEMM microbenchmark over the Llama-3-8B/70B stage shapes: achieved TFLOP/s and weight GB/s vs
the measured peaks (MEASURED_PEAKS.json)."""
import ctypes as C
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2501_14784_b200._native import check, lib  # noqa: E402

peaks = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))
HBM, TF = peaks["hbm_gbs"], peaks["bf16_tflops"]
shapes = {"qkv8b": (6144, 4096), "o8b": (4096, 4096), "gu8b": (28672, 4096), "down8b": (4096, 14336),
          "lm": (128256, 4096), "gu70b": (57344, 8192), "qkv70b": (10240, 8192), "o70b": (8192, 8192),
          "down70b": (8192, 28672)}
Ts = [int(x) for x in sys.argv[1].split(",")] if len(sys.argv) > 1 else [1, 16, 64, 128, 256, 384, 512]
MC = [int(x) for x in sys.argv[2].split(",")] if len(sys.argv) > 2 else [0]
only = sys.argv[3].split(",") if len(sys.argv) > 3 else None
res = []
for name, (N, K) in shapes.items():
  if only and name not in only:
    continue
  for mc in MC:
    for T in Ts:
        ms = C.c_float(0)
        check(lib.ds_dbg_gemm_bench(T, N, K, 0, 20, mc, C.byref(ms)))
        s = ms.value / 1e3
        fl = 2.0 * T * N * K
        by = 2.0 * N * K + 2.0 * T * K + 2.0 * T * N
        roof = max(fl / (TF * 1e12), by / (HBM * 1e9))
        res.append(dict(shape=name, mc=mc, T=T, us=round(ms.value * 1e3, 1), tflops=round(fl / s / 1e12, 1),
                        gbs=round(by / s / 1e9, 0), roof_frac=round(roof / s, 3)))
        print(json.dumps(res[-1]), flush=True)
json.dump(res, open(os.path.join(ROOT, "gpurun_out", "gemm_bench.json"), "w"))
