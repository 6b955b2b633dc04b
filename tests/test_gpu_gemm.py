"""tcgen05 GEMM parity against an fp32 numpy reference of the same bf16 operands."""
import ctypes as C

import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def _run(T, N, K, epi=0, splits=0, seed=0):
    from paper_2501_14784_b200 import _native as nat
    from paper_2501_14784_b200.bf16 import from_bf16, to_bf16
    rng = np.random.default_rng(seed)
    x = to_bf16(rng.standard_normal((T, K)).astype(np.float32))
    w = to_bf16((rng.standard_normal((N, K)) / np.sqrt(K)).astype(np.float32))
    resid = to_bf16(rng.standard_normal((T, N)).astype(np.float32))
    ref = from_bf16(x).astype(np.float64) @ from_bf16(w).astype(np.float64).T
    out = np.zeros((T, N), dtype=np.float32 if epi == 2 else np.uint16)
    nat.check(nat.lib.ds_dbg_gemm(x.ctypes.data, w.ctypes.data, T, N, K, epi,
                                  resid.ctypes.data if epi == 1 else None, splits,
                                  out.ctypes.data))
    if epi == 1:
        ref = from_bf16(resid) + from_bf16(to_bf16(ref.astype(np.float32)))
    got = out if epi == 2 else from_bf16(out)
    return got.astype(np.float64), ref


@pytest.mark.parametrize("T", [1, 7, 16, 33, 128, 256, 300, 512, 777])
def test_gemm_shapes(T):
    got, ref = _run(T, 512, 256)
    tol = 2e-2 * np.abs(ref).max() + 1e-3
    assert np.abs(got - ref).max() <= tol


@pytest.mark.parametrize("epi", [0, 1, 2])
@pytest.mark.parametrize("clusters", [1, 3, 5, 0])
def test_gemm_epilogues_and_partitions(epi, clusters):
    # clusters = cap on 2-CTA clusters: 1 -> one cluster owns whole tiles; 3, 5 -> data-parallel
    # rounds plus a stream-K remainder whose split tiles the last-arriving CTA finishes; 0 -> all
    # SMs (every tile split across several clusters)
    got, ref = _run(64, 256 * 3, 1024, epi=epi, splits=clusters, seed=3)
    tol = (1e-4 if epi == 2 else 2e-2) * np.abs(ref).max() + 1e-3
    assert np.abs(got - ref).max() <= tol


@pytest.mark.parametrize("T,clusters", [(600, 2), (777, 0), (300, 7)])
def test_gemm_two_token_blocks_stream_k(T, clusters):
    got, ref = _run(T, 1024, 512, epi=1, splits=clusters, seed=T)
    assert np.abs(got - ref).max() <= 2e-2 * np.abs(ref).max() + 1e-3


def test_gemm_llama8b_qkv_shape():
    got, ref = _run(200, 6144, 4096, seed=5)
    assert np.abs(got - ref).max() <= 2e-2 * np.abs(ref).max()


@pytest.mark.parametrize("N,K", [(512, 256), (256, 256), (1536, 256), (256, 768), (128256, 256)])
@pytest.mark.parametrize("T", [1, 17, 300])
def test_gemm_tiny_model_shapes(N, K, T):
    got, ref = _run(T, N, K, epi=2 if N == 128256 else 1, seed=N + T)
    assert np.abs(got - ref).max() <= 2e-2 * np.abs(ref).max() + 1e-3


def _silu_ref(acc):
    """h[t, 16G + j] from the 16-row interleaved gate/up accumulator (EPI_SILU)."""
    from paper_2501_14784_b200.bf16 import from_bf16, to_bf16
    T, N = acc.shape
    a = acc.reshape(T, N // 32, 2, 16)
    g = from_bf16(to_bf16(a[:, :, 0, :].astype(np.float32))).astype(np.float64)
    u = from_bf16(to_bf16(a[:, :, 1, :].astype(np.float32))).astype(np.float64)
    sg = from_bf16(to_bf16((g / (1.0 + np.exp(-g))).astype(np.float32))).astype(np.float64)
    return (sg * u).reshape(T, N // 2)


@pytest.mark.parametrize("T,clusters", [(1, 0), (33, 0), (180, 0), (300, 0), (64, 3), (40, 1)])
def test_gemm_silu_epilogue(T, clusters):
    from paper_2501_14784_b200 import _native as nat
    from paper_2501_14784_b200.bf16 import from_bf16, to_bf16
    N, K = 2048, 512
    rng = np.random.default_rng(T)
    x = to_bf16(rng.standard_normal((T, K)).astype(np.float32))
    w = to_bf16((rng.standard_normal((N, K)) / np.sqrt(K)).astype(np.float32))
    acc = from_bf16(x).astype(np.float64) @ from_bf16(w).astype(np.float64).T
    ref = _silu_ref(acc)
    out = np.zeros((T, N // 2), dtype=np.uint16)
    nat.check(nat.lib.ds_dbg_gemm(x.ctypes.data, w.ctypes.data, T, N, K, 3, None, clusters,
                                  out.ctypes.data))
    got = from_bf16(out).astype(np.float64)
    assert np.abs(got - ref).max() <= 2e-2 * np.abs(ref).max() + 1e-3



@pytest.mark.parametrize("T", [600, 1100])
def test_gemm_wide_multi_token_blocks(T):
    # wide GEMM (>= one wave of 256-row pair tiles) above 512 tokens: 256-token blocks, tile
    # order token-block-fastest, data-parallel rounds + remainder
    got, ref = _run(T, 19456, 256, epi=1, seed=T)
    assert np.abs(got - ref).max() <= 2e-2 * np.abs(ref).max() + 1e-3


@pytest.mark.parametrize("T", [700])
def test_gemm_wide_silu_multi_token_blocks(T):
    from paper_2501_14784_b200 import _native as nat
    from paper_2501_14784_b200.bf16 import from_bf16, to_bf16
    N, K = 19456, 256
    rng = np.random.default_rng(T)
    x = to_bf16(rng.standard_normal((T, K)).astype(np.float32))
    w = to_bf16((rng.standard_normal((N, K)) / np.sqrt(K)).astype(np.float32))
    acc = from_bf16(x).astype(np.float64) @ from_bf16(w).astype(np.float64).T
    ref = _silu_ref(acc)
    out = np.zeros((T, N // 2), dtype=np.uint16)
    nat.check(nat.lib.ds_dbg_gemm(x.ctypes.data, w.ctypes.data, T, N, K, 3, None, 0, out.ctypes.data))
    got = from_bf16(out).astype(np.float64)
    assert np.abs(got - ref).max() <= 2e-2 * np.abs(ref).max() + 1e-3


def _run_norm(T, N, K, N2, seed=0):
    from paper_2501_14784_b200 import _native as nat
    from paper_2501_14784_b200.bf16 import from_bf16, to_bf16
    rng = np.random.default_rng(seed)
    x = to_bf16(rng.standard_normal((T, K)).astype(np.float32))
    w1 = to_bf16((rng.standard_normal((N, K)) / np.sqrt(K)).astype(np.float32))
    w2 = to_bf16((rng.standard_normal((N2, N)) / np.sqrt(N)).astype(np.float32))
    resid = to_bf16(rng.standard_normal((T, N)).astype(np.float32))
    ox = np.zeros((T, N), dtype=np.uint16)
    oy = np.zeros((T, N2), dtype=np.uint16)
    fused = C.c_int32(0)
    eps = 1e-5
    nat.check(nat.lib.ds_dbg_gemm_norm(x.ctypes.data, w1.ctypes.data, T, N, K, resid.ctypes.data,
                                       w2.ctypes.data, N2, eps, ox.ctypes.data, oy.ctypes.data,
                                       C.byref(fused)))
    ref = from_bf16(x).astype(np.float64) @ from_bf16(w1).astype(np.float64).T
    ref_x = from_bf16(resid) + from_bf16(to_bf16(ref.astype(np.float32)))
    gx = from_bf16(ox).astype(np.float64)
    # RMSNorm (unit gains) of the x the producer wrote, then the consumer GEMM, in float64
    r = 1.0 / np.sqrt((gx ** 2).sum(1) / N + eps)
    y_ref = (gx * r[:, None]) @ from_bf16(w2).astype(np.float64).T
    return gx, ref_x, from_bf16(oy).astype(np.float64), y_ref, fused.value


# RMSNorm split across a residual GEMM and its consumer (RowNorm): k-split producers (o / down at
# 8B, T <= 256) and whole-tile producers (token-split o, prefill shapes) feeding whole-tile,
# stream-K and k-split consumers (q/k/v, gate/up shapes); a 70B-sized producer at T = 180 leaves
# k-range planes, so that pair falls back to the RMSNorm kernel
@pytest.mark.parametrize("T,N,K,N2,want_fused", [
    (1, 4096, 4096, 4096, 1), (37, 4096, 4096, 28672, 1), (180, 4096, 4096, 28672, 1),
    (256, 4096, 14336, 6144, 0), (300, 4096, 4096, 6144, 1), (1000, 4096, 4096, 28672, 1),
    (600, 8192, 8192, 10240, 1), (180, 8192, 8192, 28672, 0),
])
def test_gemm_rownorm_pair(T, N, K, N2, want_fused):
    gx, ref_x, gy, y_ref, fused = _run_norm(T, N, K, N2, seed=T + N)
    assert fused == want_fused
    assert np.abs(gx - ref_x).max() <= 2e-2 * np.abs(ref_x).max() + 1e-3
    assert np.abs(gy - y_ref).max() <= 2e-2 * np.abs(y_ref).max() + 1e-3
