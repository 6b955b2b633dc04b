#!/bin/bash
# N=1 bench A/B of the prompt-attention kernels on one box (DS_ATTN_PROMPT 2 vs 3), twice each
mkdir -p gpurun_out
for rep in 1 2; do for v in 3 2; do
  DS_ATTN_PROMPT=$v timeout 300 python bench.py --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/ab_p${v}_$rep.json 2> gpurun_out/ab_p${v}_$rep.err
  echo "prompt=$v rep=$rep rc=$?"; python -c "import json;d=json.load(open('gpurun_out/ab_p${v}_$rep.json'));print(d['value'],d['ms_per_step'],d['roofline']['by_kind']['attention'])"
done; done
