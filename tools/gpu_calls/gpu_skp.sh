#!/bin/bash
# Stream-K pieces per remainder tile (DS_GEMM_SKP; 0 = uncapped) on the stage GEMM shapes where
# data-parallel rounds leave a remainder (wide GEMMs at T <= 128): 70B gate/up, 8B gate/up, LM head.
mkdir -p gpurun_out
for v in 0 2 4 8; do
  DS_GEMM_SKP=$v timeout 120 python tools/gemm_bench.py 1,16,49,64,96,128 0 gu70b,gu8b,lm > gpurun_out/skp_$v.jsonl 2> gpurun_out/skp_$v.err
done
python - <<'PY'
import json
res = {}
for v in (0, 2, 4, 8):
    for l in open(f"gpurun_out/skp_{v}.jsonl"):
        try: d = json.loads(l)
        except Exception: continue
        res.setdefault((d["shape"], d["T"]), {})[v] = (d["us"], d["roof_frac"])
for k, r in res.items():
    print(k[0], "T", k[1], "  ".join(f"skp={v}: {u} us ({f})" for v, (u, f) in r.items()))
PY
