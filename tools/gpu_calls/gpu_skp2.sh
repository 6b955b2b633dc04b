#!/bin/bash
# DS_GEMM_SKP 8 / 16 at T <= 128, and stream-K remainders with the cap above 128 tokens
# (DS_GEMM_WHOLE=0) against the whole-tile remainder (default there).
mkdir -p gpurun_out
run() { # tag env...
  tag=$1; shift
  env "$@" timeout 120 python tools/gemm_bench.py $T 0 gu70b,gu8b,lm > gpurun_out/skp2_$tag.jsonl 2> gpurun_out/skp2_$tag.err
}
T=1,49,128 run s8 DS_GEMM_SKP=8
T=1,49,128 run s16 DS_GEMM_SKP=16
T=160,180,256 run whole DS_GEMM_SKP=8
T=160,180,256 run sk8 DS_GEMM_SKP=8 DS_GEMM_WHOLE=0
T=160,180,256 run sk16 DS_GEMM_SKP=16 DS_GEMM_WHOLE=0
T=160,180,256 run sk4 DS_GEMM_SKP=4 DS_GEMM_WHOLE=0
python - <<'PY'
import json
res = {}
for v in ("s8", "s16", "whole", "sk8", "sk16", "sk4"):
    for l in open(f"gpurun_out/skp2_{v}.jsonl"):
        try: d = json.loads(l)
        except Exception: continue
        res.setdefault((d["shape"], d["T"]), {})[v] = (d["us"], d["roof_frac"])
for k, r in res.items():
    print(k[0], "T", k[1], "  ".join(f"{v}: {u} us ({f})" for v, (u, f) in r.items()))
PY
