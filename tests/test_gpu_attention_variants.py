"""The TMA-staged attention kernels (attn_decode_tma_kernel, attn_prompt_tma_kernel: K/V tiles by
cp.async.bulk.tensor with 128-byte swizzle) compute exactly what the cp.async-staged kernels do
(same MMAs in the same order): the stage output must be bit-identical across the variants."""
import os
import subprocess
import sys

import numpy as np
import pytest

from paper_2501_14784_b200 import n_devices

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
pytestmark = [pytest.mark.gpu, pytest.mark.skipif(n_devices() < 1, reason="needs a GPU")]


def _run(tmp_path, decode, prompt):
    out = str(tmp_path / f"out_{decode}_{prompt}.bin")
    env = dict(os.environ, DS_ATTN_DECODE=str(decode), DS_ATTN_PROMPT=str(prompt))
    subprocess.run([sys.executable, os.path.join(ROOT, "tests", "attn_variant_run.py"), out, ROOT],
                   check=True, env=env, timeout=300)
    return np.fromfile(out, dtype=np.uint16)


def test_tma_attention_bit_identical_to_cp_async(tmp_path):
    tma = _run(tmp_path, 3, 2)
    ref = _run(tmp_path, 2, 1)
    assert tma.size == ref.size > 0
    f = (tma.astype(np.uint32) << 16).view(np.float32)
    assert np.isfinite(f).all()
    assert np.array_equal(tma, ref)


def test_tcgen05_prompt_attention_matches(tmp_path):
    """The tcgen05 chunked-prefill kernel (DS_ATTN_PROMPT=3: S and O accumulated in TMEM, P through
    shared memory, 128-row query blocks) agrees with the mma.sync kernels within bf16 rounding
    (different accumulation order, not bit-identical)."""
    tc = _run(tmp_path, 3, 3)
    ref = _run(tmp_path, 3, 2)
    a = (tc.astype(np.uint32) << 16).view(np.float32).reshape(-1, 4096)
    b = (ref.astype(np.uint32) << 16).view(np.float32).reshape(-1, 4096)
    assert np.isfinite(a).all()
    err = np.abs(a - b).max(axis=1)
    scale = np.abs(b).max(axis=1)
    assert np.all(err <= 0.02 * scale), float((err / scale).max())
