#!/usr/bin/env python3
"""Summarise tools/gpu_calls/gpu_70b_attn.sh's ncu launch list (cold-cache, serialised launches) into
per-kind time, DRAM bytes, and fractions of the measured peaks at Llama-3-70B stage shapes.
Algorithmic bytes: weights + bf16 activations in/out (GEMMs); K and V of every row's context
once + q/o (decode attention). Usage: summarize_cal70.py launches.csv [peaks.json]"""
import collections
import csv
import json
import sys

D, NH, NKV, DH, FF = 8192, 64, 8, 128, 28672
CTX = 1024 + 1                     # decode rows at position 1024 attend over 1025 tokens
CONFIGS = [("decode T=49 ctx=1024", 49), ("decode T=256 ctx=1024", 256), ("prefill T=3840 (one prompt)", 3840)]
STEPS, LAYERS = 5, 10              # 2 warm-ups + 3 reps per config, 10-layer stage
GEMMS = [("gemm_qkv", (NH + 2 * NKV) * DH, D), ("gemm_o", D, NH * DH),
         ("gemm_gate_up", 2 * FF, D), ("gemm_down", D, FF)]


def main():
    rows = [r for r in csv.reader(open(sys.argv[1])) if len(r) == 15 and r[0] != "ID"]
    peaks = json.load(open(sys.argv[2])) if len(sys.argv) > 2 else {}
    bw = peaks.get("hbm_gbs", 6548.5)
    # kernels timed alone (serialised ncu launches): the burst tensor peak, per B200_PROFILING
    tf = peaks.get("bf16_tflops", 1647.8)
    launches = collections.OrderedDict()
    for r in rows:
        d = launches.setdefault(int(r[0]), {"name": r[4]})
        d[r[12]] = float(r[14].replace(",", ""))
    seq = list(launches.values())
    per = len(seq) // len(CONFIGS)
    out = []
    for ci, (label, T) in enumerate(CONFIGS):
        acc = collections.defaultdict(lambda: [0.0, 0.0, 0.0, 0.0, 0])  # ns, dram B, alg B, flops, n
        gi = 0
        for L in seq[ci * per:(ci + 1) * per]:
            nm = L["name"]
            ns = L["gpu__time_duration.sum"]
            dram = L["dram__bytes_read.sum"] + L["dram__bytes_write.sum"]
            if "gemm_tc" in nm:
                kind, N, K = GEMMS[gi % 4]
                gi += 1
                nout = N // 2 if kind == "gemm_gate_up" else N
                alg, fl = 2.0 * N * K + 2.0 * T * K + 2.0 * T * nout, 2.0 * T * N * K
            elif "attn_decode" in nm:
                kind = "attention_decode"
                alg = T * CTX * NKV * DH * 2 * 2 + 2 * 2.0 * T * NH * DH
                fl = 4.0 * NH * DH * CTX * T
            elif "attn_prompt" in nm:
                kind = "attention_prompt"
                alg = 2 * T * NKV * DH * 2 + 2 * 2.0 * T * NH * DH
                fl = 4.0 * NH * DH * (T * (T + 1) / 2)
            else:
                kind = "rope_kv"
                alg = fl = 0.0
            a = acc[kind]
            a[0] += ns; a[1] += dram; a[2] += alg; a[3] += fl; a[4] += 1
        kinds = {}
        for kind, (ns, dram, alg, fl, n) in acc.items():
            s = ns * 1e-9
            kinds[kind] = {"launches": n, "us_per_launch": round(ns / n / 1e3, 2),
                           "dram_gbs": round(dram / s / 1e9, 1),
                           "dram_frac_of_hbm": round(dram / s / 1e9 / bw, 3),
                           "alg_gbs": round(alg / s / 1e9, 1) if alg else None,
                           "alg_frac_of_hbm": round(alg / s / 1e9 / bw, 3) if alg else None,
                           "tflops": round(fl / s / 1e12, 1) if fl else None,
                           "tensor_frac": round(fl / s / 1e12 / tf, 3) if fl else None}
        out.append({"config": label, "T": T, "kinds": kinds})
    print(json.dumps({"source": sys.argv[1], "hbm_gbs": bw, "bf16_tflops_burst": tf,
                      "note": "ncu launch list: serialised, cold-cache launches (--clock-control none)",
                      "configs": out}, indent=1))


if __name__ == "__main__":
    main()
