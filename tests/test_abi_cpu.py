"""C-ABI checks that need no GPU: libdeserve_b200.so exports every function include/deserve.h
declares, and the GEMM work partition (host arithmetic of gemm_tc.cu's plan_gemm, queried through
ds_dbg_gemm_plan) follows the documented rules at the Llama-3-8B / 70B stage shapes."""
import ctypes as C
import os
import re

import pytest

from paper_2501_14784_b200 import _native as nat

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
FIELDS = ("status", "cn", "clusters", "dp_rounds", "sk_tiles", "n_sk", "ks", "planes", "defer", "tb",
          "t_blocks", "kb")
NUM_SMS = 148


def declared_functions():
    src = open(os.path.join(ROOT, "include", "deserve.h")).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    src = re.sub(r"//[^\n]*", "", src)
    pat = r"^\s*(?:const\s+)?[a-z_0-9]+\s*\**\s*\b(ds_[a-z0-9_]+)\s*\("
    return sorted(set(m.group(1) for m in re.finditer(pat, src, flags=re.M)))


def test_library_exports_every_declared_function():
    names = declared_functions()
    assert len(names) > 40 and "ds_stage_step" in names and "ds_run" in names
    lib = C.CDLL(nat.LIB_PATH)
    missing = [n for n in names if not hasattr(lib, n)]
    assert missing == []


def plan(T, N, K):
    out = (C.c_int32 * 12)()
    nat.check(nat.lib.ds_dbg_gemm_plan(T, N, K, out))
    return dict(zip(FIELDS, list(out)))


# (N, K) of the stage GEMMs: q/k/v, o, gate/up (interleaved), down, LM head
SHAPES = {"qkv8b": (6144, 4096), "o8b": (4096, 4096), "gu8b": (28672, 4096), "down8b": (4096, 14336),
          "lm": (128256, 4096), "qkv70b": (10240, 8192), "o70b": (8192, 8192), "gu70b": (57344, 8192),
          "down70b": (8192, 28672)}


def test_gemm_plan_needs_a_valid_shape():
    out = (C.c_int32 * 12)()
    assert nat.lib.ds_dbg_gemm_plan(0, 4096, 4096, out) != 0
    assert nat.lib.ds_dbg_gemm_plan(16, 4000, 4096, out) != 0  # N not a multiple of 128


@pytest.mark.parametrize("T", [1, 49, 128])
def test_stream_k_remainder_pieces_capped(T):
    """70B gate/up: 224 pair tiles = 3 data-parallel rounds over 74 clusters + 2 remainder tiles,
    each split into at most 8 stream-K pieces (DS_GEMM_SKP; profiles/r02_gemm_skp.txt)."""
    p = plan(T, *SHAPES["gu70b"])
    assert (p["cn"], p["clusters"], p["dp_rounds"], p["sk_tiles"]) == (2, 74, 3, 2)
    assert p["n_sk"] == 16


@pytest.mark.parametrize("T", [180, 256])
def test_remainder_tiles_whole_above_128_tokens(T):
    p = plan(T, *SHAPES["gu70b"])
    assert p["dp_rounds"] == 3 and p["n_sk"] == p["sk_tiles"] == 2
    p = plan(T, *SHAPES["gu8b"])
    assert p["dp_rounds"] == 1 and p["n_sk"] == p["sk_tiles"] == 38


def test_8b_decode_partitions():
    """The launch sequence DESIGN.md section 4 describes at a 180-row decode circuit: o and down
    as 4-way k-split clusters (DSMEM reduction), q/k/v as k-range planes summed by the RoPE
    kernel, gate/up one data-parallel round plus whole remainder tiles."""
    o, down, qkv, gu = (plan(180, *SHAPES[k]) for k in ("o8b", "down8b", "qkv8b", "gu8b"))
    assert o["ks"] == 4 and down["ks"] == 4
    assert qkv["ks"] == 1 and qkv["planes"] == 3 and qkv["defer"] == 1
    assert gu["ks"] == 1 and gu["planes"] == 0 and gu["dp_rounds"] == 1
    p = plan(16, *SHAPES["gu8b"])  # <= 128 tokens: the remainder is stream-K, <= 2 pieces a tile
    assert p["sk_tiles"] == 38 and p["n_sk"] == 74


@pytest.mark.parametrize("name", sorted(SHAPES))
@pytest.mark.parametrize("T", [1, 16, 49, 128, 180, 256, 300, 512, 1024, 4096, 16384])
def test_partition_invariants(name, T):
    N, K = SHAPES[name]
    p = plan(T, N, K)
    assert p["status"] == 0 and p["kb"] == K // 64
    ctas = p["clusters"] * p["cn"] * max(1, p["ks"])
    assert 1 <= ctas <= NUM_SMS
    assert p["tb"] * p["t_blocks"] >= T and p["tb"] <= 512
    if p["ks"] > 1:  # k-split clusters: one tile per cluster, no stream-K
        assert p["sk_tiles"] == 0 and p["dp_rounds"] == 0
        return
    tiles = p["t_blocks"] * (N // 128) // p["cn"]
    if p["dp_rounds"] > 0:  # whole rounds cover all but the stream-K remainder
        assert p["dp_rounds"] * p["clusters"] + p["sk_tiles"] == tiles
    assert p["n_sk"] <= p["sk_tiles"] * p["kb"]  # no empty stream-K range
    if p["dp_rounds"] > 0 and p["sk_tiles"] > 0:
        assert p["n_sk"] <= 8 * p["sk_tiles"]
