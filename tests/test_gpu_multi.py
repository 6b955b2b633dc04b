"""One process per GPU (torchrun) with NCCL hops must produce exactly the tokens of the
in-process pipeline on the same schedule (same kernels, same rows; only the transport differs)."""
import json
import os
import subprocess
import sys

import pytest

from paper_2501_14784_b200 import n_devices
from paper_2501_14784_b200 import pipeline as pl

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
pytestmark = [pytest.mark.gpu, pytest.mark.skipif(n_devices() < 2, reason="needs 2 GPUs")]


def test_nccl_ring_matches_in_process():
    out = os.path.join(ROOT, "gpurun_out", "nccl_tokens_2.json")
    if os.path.exists(out):
        os.remove(out)
    os.makedirs(os.path.dirname(out), exist_ok=True)
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node", "2",
           "--master-addr", "127.0.0.1", "--master-port", "29531",
           os.path.join(ROOT, "tools", "nccl_pipeline.py"), "tiny_2stage.json", "40"]
    subprocess.run(cmd, check=True, timeout=240)
    nccl_tokens = json.load(open(out))
    cdir = os.path.join(ROOT, "configs")
    r = pl.gpu_run_config(open(os.path.join(cdir, "tiny_2stage.json")).read(), cdir,
                          collect_tokens=True, max_circuits=40, n_devices=1)
    assert r["tokens"] == nccl_tokens
