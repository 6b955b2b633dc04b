#!/bin/bash
# A/B of two builds of the library on one box (abso/lib_old.so vs abso/lib_new.so): N=1 bench
# alternating, twice each, plus the narrow-GEMM shapes.
mkdir -p gpurun_out
L=paper_2501_14784_b200/libdeserve_b200.so
for rep in 1 2; do for v in old new; do
  cp abso/lib_$v.so $L
  timeout 600 python bench.py --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/ab_$v$rep.json 2> gpurun_out/ab_$v$rep.err
  python -c "import json;d=json.load(open('gpurun_out/ab_$v$rep.json'));print('$v$rep',d['value'],d['clocks']['sm_mhz'],{k:v['ms'] for k,v in d['roofline']['by_kind'].items()})"
done; done
for v in old new; do cp abso/lib_$v.so $L; echo $v; bash tools/gemm_quick.sh 16,64,180,256 o8b,gu8b,down8b 2>&1; done
rm -f gpurun_out/bench_n1.trace
