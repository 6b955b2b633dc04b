#!/bin/bash
# One-GPU measurement pass (run under gpurun): GPU tests, the N=1 bench line, the reference arm,
# the GEMM shape sweep and an ncu launch list of a mid-schedule window of the bench step.
# Outputs under gpurun_out/<tag>_*.
tag=${1:-r02}
mkdir -p gpurun_out
python -m pytest tests -m gpu -q -x -p no:cacheprovider > gpurun_out/${tag}_gputests.log 2>&1
echo "gpu tests rc=$?"; tail -3 gpurun_out/${tag}_gputests.log
python bench.py --steps 3 --warmup 3 > gpurun_out/${tag}_bench_n1.json 2> gpurun_out/${tag}_bench_n1.err
echo "bench rc=$?"; tail -c 400 gpurun_out/${tag}_bench_n1.json
python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/${tag}_bench_ref.json 2> gpurun_out/${tag}_bench_ref.err
echo "ref arm rc=$?"; tail -c 300 gpurun_out/${tag}_bench_ref.json
bash tools/gemm_quick.sh 16,64,128,180,256,512,1024,4096,8192 > gpurun_out/${tag}_gemm.txt 2>&1; python tools/gemm_bench.py 256,1024,4096,8192 0 gu70b > gpurun_out/${tag}_gemm70b.txt 2>&1
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none \
    --cache-control none -s 60000 -c 6000 --csv --log-file gpurun_out/${tag}_launches.csv \
    python tools/step_driver.py --circuits 761 > gpurun_out/${tag}_ncu.log 2>&1
echo "ncu rc=$?"
python tools/summarize_ncu.py launches gpurun_out/${tag}_launches.csv > gpurun_out/${tag}_launch_shares.csv 2>&1
head -20 gpurun_out/${tag}_launch_shares.csv
