#!/bin/bash
# Remainder rule A/B (new default: capped stream-K pieces, whole remainders only when they fill
# more than half the clusters; old: DS_GEMM_WHOLE=2 DS_GEMM_SKP=0) on every stage GEMM shape,
# then the GPU suite + smoke() with the new default, then the N=1 bench new vs old.
mkdir -p gpurun_out
S=gu70b,qkv70b,o70b,down70b,gu8b,qkv8b,o8b,down8b,lm
timeout 150 python tools/gemm_bench.py 1,49,128,180,256,1024,4096 0 $S > gpurun_out/skp3_new.jsonl 2> gpurun_out/skp3_new.err
DS_GEMM_WHOLE=2 DS_GEMM_SKP=0 timeout 150 python tools/gemm_bench.py 1,49,128,180,256,1024,4096 0 $S > gpurun_out/skp3_old.jsonl 2> gpurun_out/skp3_old.err
python - <<'PY'
import json
res = {}
for v in ("old", "new"):
    for l in open(f"gpurun_out/skp3_{v}.jsonl"):
        try: d = json.loads(l)
        except Exception: continue
        res.setdefault((d["shape"], d["T"]), {})[v] = (d["us"], d["roof_frac"])
for k, r in res.items():
    flag = "" if "old" not in r or "new" not in r else ("  <-- changed %+.1f%%" % (100 * (r["new"][0] / r["old"][0] - 1)) if abs(r["new"][0] / r["old"][0] - 1) > 0.02 else "")
    print(k[0], "T", k[1], "  ".join(f"{v}: {u} us ({f})" for v, (u, f) in r.items()), flag)
PY
timeout 300 python -m pytest tests -m gpu -q -x -p no:cacheprovider > gpurun_out/skp3_gputests.log 2>&1
echo "gpu tests rc=$?"; grep -E 'passed|failed|Error' gpurun_out/skp3_gputests.log | tail -5
timeout 120 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/skp3_smoke.log 2>&1; echo "smoke rc=$?"; tail -1 gpurun_out/skp3_smoke.log
timeout 200 python bench.py --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/skp3_bench_new.json 2> gpurun_out/skp3_bench_new.err
python -c "import json;d=json.load(open('gpurun_out/skp3_bench_new.json'));print('new',d['value'],d['clocks']['sm_mhz'],{k:round(v['ms'],1) for k,v in d['roofline']['by_kind'].items()})"
DS_GEMM_WHOLE=2 DS_GEMM_SKP=0 timeout 200 python bench.py --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/skp3_bench_old.json 2> gpurun_out/skp3_bench_old.err
python -c "import json;d=json.load(open('gpurun_out/skp3_bench_old.json'));print('old',d['value'],d['clocks']['sm_mhz'],{k:round(v['ms'],1) for k,v in d['roofline']['by_kind'].items()})"
rm -f gpurun_out/bench_n1.trace
