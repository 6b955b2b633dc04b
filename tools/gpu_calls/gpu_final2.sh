#!/bin/bash
# End-of-round one-GPU pass: GPU suite, smoke(), and ncu --set full of the final tcgen05 prompt
# kernel on one layer of a 3840-token prompt (Llama-3-8B).
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/r02h_gputests.log 2>&1
echo "gpu tests rc=$?"; tail -3 gpurun_out/r02h_gputests.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r02h_smoke.log 2>&1; echo "smoke rc=$?"; tail -1 gpurun_out/r02h_smoke.log
timeout 300 ncu --set full --import-source on --clock-control none -k regex:attn_prompt_tc --launch-skip 40 --launch-count 1 -o gpurun_out/r02h_prompt_tc -f python tools/calibrate_stage.py --decode "" --prefill 3840 --reps 1 > gpurun_out/r02h_ncu.log 2>&1
echo "ncu rc=$?"; python tools/summarize_ncu.py full gpurun_out/r02h_prompt_tc.ncu-rep > gpurun_out/r02h_prompt_tc.csv 2>&1; cat gpurun_out/r02h_prompt_tc.csv
