#!/bin/bash
# Final one-GPU pass: the whole GPU test suite, smoke(), the N=1 bench line (with cpu_baseline),
# the reference arm, and the ncu launch list of a mid-schedule window (kernel shares).
tag=${1:-r02f}
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/${tag}_gputests.log 2>&1
echo "gpu tests rc=$?"; tail -4 gpurun_out/${tag}_gputests.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/${tag}_smoke.log 2>&1; echo "smoke rc=$?"; tail -2 gpurun_out/${tag}_smoke.log
timeout 600 python bench.py --steps 3 --warmup 3 > gpurun_out/${tag}_bench_n1.json 2> gpurun_out/${tag}_bench_n1.err
echo "bench rc=$?"; python -c "import json;d=json.load(open('gpurun_out/${tag}_bench_n1.json'));print(d['value'],d['ms_per_step'],d['e2e']['value'],d['roofline']['frac'],d['clocks'],{k:v['ms'] for k,v in d['roofline']['by_kind'].items()})"
timeout 600 python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/${tag}_bench_ref.json 2> gpurun_out/${tag}_bench_ref.err
echo "ref arm rc=$?"; tail -c 300 gpurun_out/${tag}_bench_ref.json
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none \
    --cache-control none -s 60000 -c 6000 --csv --log-file gpurun_out/${tag}_launches.csv \
    python tools/step_driver.py --circuits 761 > gpurun_out/${tag}_ncu.log 2>&1
echo "ncu rc=$?"
python tools/summarize_ncu.py launches gpurun_out/${tag}_launches.csv > gpurun_out/${tag}_launch_shares.csv 2>&1
head -12 gpurun_out/${tag}_launch_shares.csv
rm -f gpurun_out/bench_n1.trace
