// Paged causal GQA attention over the stage's KV pages on tensor cores (mma.sync m16n8k16 bf16,
// fp32 accumulate), FlashAttention-2 style with an online softmax in the log2 domain.
//
// Two kernels per layer:
//  * prompt blocks (attn_prompt_kernel): up to QP = 64/G consecutive prompt positions of one
//    request (chunked prefill, reference begin_circuit sim.cpp:386-407); the G = n_h / n_kv query
//    heads of a KV head share every staged 64-token K/V tile (a 256-token page never straddled),
//    so the request's KV is read once per block; 8 warps = 4 row groups x 2 tile parities.
//  * decode rows (attn_decode_t_kernel, attn_decode_kernel for G > 8): one row x KV head per CTA,
//    per-warp cp.async rings over 16-token chunks, operand-swapped GQA MMAs.
// Context splits (flash-decoding) when rows are few; the last CTA of each (row / block, KV head)
// merges the (o, m, l) partials in split order.
//
// HBM roofline: each (row or block, kv head) reads its request's KV once: ctx * d_head * 2 (K,V)
// * 2 B per kv head.
#include <cuda.h>
#include <stdlib.h>

#include <algorithm>

#include "common.cuh"
#include "kernels.h"

namespace ds {

constexpr int kTile = 64;
constexpr int kAttnWarps = 4;

DS_DEVICE void cp_async16(void* smem, const void* gmem) {
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(smem_u32(smem)), "l"(gmem) : "memory");
}
DS_DEVICE void cp_async_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
template <int N>
DS_DEVICE void cp_async_wait() {
    asm volatile("cp.async.wait_group %0;" ::"n"(N) : "memory");
}
DS_DEVICE void ldsm_x4(uint32_t addr, uint32_t& r0, uint32_t& r1, uint32_t& r2, uint32_t& r3) {
    asm volatile("ldmatrix.sync.aligned.m8n8.x4.shared.b16 {%0,%1,%2,%3}, [%4];"
                 : "=r"(r0), "=r"(r1), "=r"(r2), "=r"(r3)
                 : "r"(addr));
}
DS_DEVICE void ldsm_x4_t(uint32_t addr, uint32_t& r0, uint32_t& r1, uint32_t& r2, uint32_t& r3) {
    asm volatile("ldmatrix.sync.aligned.m8n8.x4.trans.shared.b16 {%0,%1,%2,%3}, [%4];"
                 : "=r"(r0), "=r"(r1), "=r"(r2), "=r"(r3)
                 : "r"(addr));
}
DS_DEVICE void mma16816(float* c, const uint32_t* a, uint32_t b0, uint32_t b1) {
    asm volatile(
        "mma.sync.aligned.m16n8k16.row.col.f32.bf16.bf16.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, "
        "{%0,%1,%2,%3};"
        : "+f"(c[0]), "+f"(c[1]), "+f"(c[2]), "+f"(c[3])
        : "r"(a[0]), "r"(a[1]), "r"(a[2]), "r"(a[3]), "r"(b0), "r"(b1));
}

// ------------------------------------------------------------------ prompt blocks ----
// One (prompt query block, KV head, context split) per CTA of 8 warps: warp w owns q rows
// 16*(w%4).. of the block (<= 64 = positions x G heads) and the tiles of parity w/4, so the two
// halves of the CTA walk alternate 64-token K/V tiles at the same time (half the serial chain of
// a long prompt chunk) and merge their softmax states through shared memory at the end. Tile
// pairs are double-buffered with cp.async.
constexpr int kPromptWarps = 8;

template <int DH>
struct PromptSmem {
    __nv_bfloat16 k[2][2][kTile][DH + 8];  // [pair buffer][parity]
    __nv_bfloat16 v[2][2][kTile][DH + 8];
    __nv_bfloat16 q[64][DH + 8];           // the block's query rows (r = position * G + head)
};

// blocks: [n_blocks][3] = (first row t0, n positions, unused)
template <int DH>
__global__ void __launch_bounds__(kPromptWarps * 32)
attn_prompt_kernel(const __nv_bfloat16* __restrict__ q, int n_h, const int32_t* __restrict__ row_pos,
                   const int32_t* __restrict__ row_page_off, const int32_t* __restrict__ flat_pages,
                   const int32_t* __restrict__ blocks, KvLayout kv, int layer, int splits, int stride,
                   __nv_bfloat16* __restrict__ o, float* __restrict__ ws, int* __restrict__ counters,
                   L2Prefetch pf) {
    pdl_launch_dependents();
    l2_prefetch_slice(pf);
    pdl_wait();
    extern __shared__ __align__(16) uint8_t attn_smem[];
    PromptSmem<DH>& sm = *reinterpret_cast<PromptSmem<DH>*>(attn_smem);
    constexpr int NT = DH / 8;   // output n-tiles
    constexpr int KS = DH / 16;  // k-steps over d_head
    constexpr int SN = kTile / 8;
    const int n_kv = kv.n_kv;
    const int G = n_h / n_kv;
    const int split = blockIdx.x % splits;
    const int kvh = (blockIdx.x / splits) % n_kv;
    const int bi = blockIdx.x / (splits * n_kv);
    const int t0 = blocks[3 * bi], npos = blocks[3 * bi + 1];
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int rg = warp & 3, par = warp >> 2;
    const int g = lane >> 2, tq = lane & 3;
    const int rows = npos * G;  // q rows of this block: r = p * G + h
    const int pos0 = row_pos[t0];
    const int last_pos = pos0 + npos - 1;
    const int n_tiles = (last_pos + kTile) / kTile;
    const int tile0 = split * n_tiles / splits, tile1 = (split + 1) * n_tiles / splits;
    const int32_t* pages = flat_pages + row_page_off[t0];

    const int r_base = rg * 16;
    const bool warp_active = r_base < rows;
    // Q rows stream into shared memory with the first K/V tiles (cp.async, 16 B per request, the
    // G heads of a position contiguous); fragments via ldmatrix once they land. S is scaled by
    // log2(e)/sqrt(d_head) after the MMA.
    uint32_t qa[KS][4];
    const float qs = rsqrtf(float(DH)) * 1.4426950408889634f;
    for (int i = threadIdx.x; i < rows * (DH / 8); i += blockDim.x) {
        const int r = i / (DH / 8), c = (i % (DH / 8)) * 8;
        cp_async16(&sm.q[r][c], q + (size_t(t0 + r / G) * n_h + kvh * G + r % G) * DH + c);
    }
    int rpos[2];
#pragma unroll
    for (int hr = 0; hr < 2; ++hr) {
        const int r = r_base + g + 8 * hr;
        rpos[hr] = r < rows ? pos0 + r / G : -1;
    }

    float m_run[2] = {-INFINITY, -INFINITY}, l_run[2] = {0.f, 0.f};
    float acc[NT][4];
#pragma unroll
    for (int j = 0; j < NT; ++j) acc[j][0] = acc[j][1] = acc[j][2] = acc[j][3] = 0.f;

    const size_t head_k = ((size_t(layer) * 2 + 0) * n_kv + kvh) * 256 * DH;
    const size_t head_v = ((size_t(layer) * 2 + 1) * n_kv + kvh) * 256 * DH;
    constexpr int CHUNKS = kTile * DH / 8;  // 16-byte chunks per K (or V) tile
    const int n_pairs = (tile1 - tile0 + 1) / 2;
    auto load_pair = [&](int pi, int buf) {
        for (int pp = 0; pp < 2; ++pp) {
            const int tile = tile0 + 2 * pi + pp;
            if (tile >= tile1) break;
            const int tok0 = tile * kTile;
            const size_t base = size_t(pages[tok0 >> 8]) * kv.page_elems + size_t(tok0 & 255) * DH;
            const __nv_bfloat16* ks = kv.pool + base + head_k;
            const __nv_bfloat16* vs = kv.pool + base + head_v;
            for (int i = threadIdx.x; i < CHUNKS; i += blockDim.x) {
                const int r = i / (DH / 8), c = (i % (DH / 8)) * 8;
                cp_async16(&sm.k[buf][pp][r][c], ks + size_t(r) * DH + c);
                cp_async16(&sm.v[buf][pp][r][c], vs + size_t(r) * DH + c);
            }
        }
        cp_async_commit();
    };

    if (n_pairs > 0) {
        load_pair(0, 0);  // commits the Q rows with the first tile pair
    } else {
        cp_async_commit();
        cp_async_wait<0>();
    }
    for (int pi = 0; pi < n_pairs; ++pi) {
        const int buf = pi & 1;
        if (pi + 1 < n_pairs) {
            load_pair(pi + 1, buf ^ 1);
            cp_async_wait<1>();
        } else {
            cp_async_wait<0>();
        }
        __syncthreads();
        if (pi == 0 && warp_active) {  // the Q rows landed with the first pair
#pragma unroll
            for (int kk = 0; kk < KS; ++kk)
                ldsm_x4(smem_u32(&sm.q[r_base + (lane & 15)][kk * 16 + (lane >> 4) * 8]), qa[kk][0],
                        qa[kk][1], qa[kk][2], qa[kk][3]);
        }
        // zero V rows past the last valid token (0 * garbage must not produce NaN)
        for (int pp = 0; pp < 2; ++pp) {
            const int tile = tile0 + 2 * pi + pp;
            if (tile >= tile1) break;
            const int valid = min(kTile, last_pos + 1 - tile * kTile);
            for (int i = threadIdx.x; i < (kTile - valid) * (DH / 8); i += blockDim.x) {
                const int r = valid + i / (DH / 8), c = (i % (DH / 8)) * 8;
                *reinterpret_cast<uint4*>(&sm.v[buf][pp][r][c]) = make_uint4(0, 0, 0, 0);
            }
        }
        __syncthreads();
        const int tile = tile0 + 2 * pi + par;
        if (warp_active && tile < tile1) {
            const int tok0 = tile * kTile;
            float s[SN][4];
#pragma unroll
            for (int j = 0; j < SN; ++j) s[j][0] = s[j][1] = s[j][2] = s[j][3] = 0.f;
            const uint32_t kbase = smem_u32(&sm.k[buf][par][0][0]);
#pragma unroll
            for (int j = 0; j < SN; ++j)
#pragma unroll
                for (int kk = 0; kk < KS; kk += 2) {
                    const int mi = lane >> 3, rr = lane & 7;
                    uint32_t b0, b1, b2, b3;
                    ldsm_x4(kbase + uint32_t(((j * 8 + rr) * (DH + 8) + kk * 16 + mi * 8) * 2), b0, b1, b2, b3);
                    mma16816(s[j], qa[kk], b0, b1);
                    mma16816(s[j], qa[kk + 1], b2, b3);
                }
            // scale, causal mask + online softmax (rows g and g+8)
            float mt[2] = {-INFINITY, -INFINITY};
#pragma unroll
            for (int j = 0; j < SN; ++j)
#pragma unroll
                for (int e = 0; e < 4; ++e) {
                    const int hr = e >> 1;
                    s[j][e] = tok0 + j * 8 + 2 * tq + (e & 1) > rpos[hr] ? -INFINITY : s[j][e] * qs;
                    mt[hr] = fmaxf(mt[hr], s[j][e]);
                }
            float alpha[2];
#pragma unroll
            for (int hr = 0; hr < 2; ++hr) {
                mt[hr] = fmaxf(mt[hr], __shfl_xor_sync(0xffffffffu, mt[hr], 1));
                mt[hr] = fmaxf(mt[hr], __shfl_xor_sync(0xffffffffu, mt[hr], 2));
                const float mn = fmaxf(m_run[hr], mt[hr]);
                alpha[hr] = mn == -INFINITY ? 1.f : exp2f(m_run[hr] - mn);
                m_run[hr] = mn;
            }
            float ls[2] = {0.f, 0.f};
            uint32_t pa[SN / 2][4];
#pragma unroll
            for (int j = 0; j < SN; ++j)
#pragma unroll
                for (int e = 0; e < 4; ++e) {
                    const int hr = e >> 1;
                    const float pv = m_run[hr] == -INFINITY ? 0.f : exp2f(s[j][e] - m_run[hr]);
                    s[j][e] = pv;
                    ls[hr] += pv;
                }
#pragma unroll
            for (int hr = 0; hr < 2; ++hr) l_run[hr] = l_run[hr] * alpha[hr] + ls[hr];  // quad-partial
#pragma unroll
            for (int j = 0; j < NT; ++j) {
                acc[j][0] *= alpha[0];
                acc[j][1] *= alpha[0];
                acc[j][2] *= alpha[1];
                acc[j][3] *= alpha[1];
            }
#pragma unroll
            for (int kk = 0; kk < SN / 2; ++kk) {
                pa[kk][0] = pack2(s[2 * kk][0], s[2 * kk][1]);
                pa[kk][1] = pack2(s[2 * kk][2], s[2 * kk][3]);
                pa[kk][2] = pack2(s[2 * kk + 1][0], s[2 * kk + 1][1]);
                pa[kk][3] = pack2(s[2 * kk + 1][2], s[2 * kk + 1][3]);
            }
            const uint32_t vbase = smem_u32(&sm.v[buf][par][0][0]);
#pragma unroll
            for (int kk = 0; kk < SN / 2; ++kk)
#pragma unroll
                for (int nt = 0; nt < NT; nt += 2) {
                    const int mi = lane >> 3, rr = lane & 7;
                    uint32_t b0, b1, b2, b3;
                    ldsm_x4_t(vbase + uint32_t(((kk * 16 + (mi & 1) * 8 + rr) * (DH + 8) + (nt + (mi >> 1)) * 8) * 2),
                              b0, b1, b2, b3);
                    mma16816(acc[nt], pa[kk], b0, b1);
                    mma16816(acc[nt + 1], pa[kk], b2, b3);
                }
        }
        __syncthreads();  // pair buffer `buf` is overwritten by the prefetch of pair pi + 2
    }

#pragma unroll
    for (int hr = 0; hr < 2; ++hr) {  // full row sums across the quad
        l_run[hr] += __shfl_xor_sync(0xffffffffu, l_run[hr], 1);
        l_run[hr] += __shfl_xor_sync(0xffffffffu, l_run[hr], 2);
    }
    // merge the odd-tile half into the even-tile half (shared memory of the idle tile buffers)
    float* red = reinterpret_cast<float*>(&sm.k[0][0][0][0]);  // [4 row groups][16 rows][DH + 2]
    if (par == 1 && warp_active) {
#pragma unroll
        for (int hr = 0; hr < 2; ++hr) {
            float* dst = red + (rg * 16 + g + 8 * hr) * (DH + 2);
#pragma unroll
            for (int nt = 0; nt < NT; ++nt) {
                dst[nt * 8 + 2 * tq] = acc[nt][2 * hr];
                dst[nt * 8 + 2 * tq + 1] = acc[nt][2 * hr + 1];
            }
            if (tq == 0) {
                dst[DH] = m_run[hr];
                dst[DH + 1] = l_run[hr];
            }
        }
    }
    __syncthreads();
    if (par == 0 && warp_active) {
#pragma unroll
    for (int hr = 0; hr < 2; ++hr) {
        const int r = r_base + g + 8 * hr;
        const float* oth = red + (rg * 16 + g + 8 * hr) * (DH + 2);
        const float m1 = oth[DH], l1 = oth[DH + 1];
        const float M = fmaxf(m_run[hr], m1);
        const float w0 = m_run[hr] == -INFINITY ? 0.f : exp2f(m_run[hr] - M);
        const float w1 = m1 == -INFINITY ? 0.f : exp2f(m1 - M);
        const float L = l_run[hr] * w0 + l1 * w1;
        if (r >= rows) continue;
        const int p = r / G, h = r % G;
        const size_t row_head = size_t(t0 + p) * n_h + kvh * G + h;
        if (splits == 1) {
            const float inv = 1.0f / L;
            __nv_bfloat16* dst = o + row_head * DH;
#pragma unroll
            for (int nt = 0; nt < NT; ++nt) {
                const int c = nt * 8 + 2 * tq;
                *reinterpret_cast<uint32_t*>(dst + c) =
                    pack2((acc[nt][2 * hr] * w0 + oth[c] * w1) * inv, (acc[nt][2 * hr + 1] * w0 + oth[c + 1] * w1) * inv);
            }
        } else {
            float* dst = ws + (row_head * stride + split) * (DH + 2);
#pragma unroll
            for (int nt = 0; nt < NT; ++nt) {
                const int c = nt * 8 + 2 * tq;
                __stcg(dst + c, acc[nt][2 * hr] * w0 + oth[c] * w1);
                __stcg(dst + c + 1, acc[nt][2 * hr + 1] * w0 + oth[c + 1] * w1);
            }
            if (tq == 0) {
                __stcg(dst + DH, M);
                __stcg(dst + DH + 1, L);
            }
        }
    }
    }
    if (splits == 1) return;
    // context splits: the last CTA of this (block, KV head) merges all splits in split order
    __threadfence();
    __syncthreads();
    __shared__ int last_cta;
    if (threadIdx.x == 0) {
        int* cnt = counters + size_t(bi) * n_kv + kvh;
        const int old = atomicAdd(cnt, 1);
        last_cta = old == splits - 1;
        if (last_cta) *cnt = 0;  // ready for the next launch
    }
    __syncthreads();
    if (!last_cta) return;
    __threadfence();
    for (int i = threadIdx.x; i < rows * DH; i += blockDim.x) {
        const int r = i / DH, dd = i % DH;
        const size_t row_head = size_t(t0 + r / G) * n_h + kvh * G + r % G;
        const float* base = ws + row_head * stride * (DH + 2);
        float M = -INFINITY;
        for (int sp = 0; sp < splits; ++sp) M = fmaxf(M, __ldcg(base + sp * (DH + 2) + DH));
        float num = 0.f, den = 0.f;
        for (int sp = 0; sp < splits; ++sp) {
            const float ms = __ldcg(base + sp * (DH + 2) + DH);
            if (ms == -INFINITY) continue;
            const float w = exp2f(ms - M);
            num += __ldcg(base + sp * (DH + 2) + dd) * w;
            den += __ldcg(base + sp * (DH + 2) + DH + 1) * w;
        }
        o[row_head * DH + dd] = f2bf(num / den);
    }
}


DS_DEVICE void fence_proxy_async_smem() { asm volatile("fence.proxy.async.shared::cta;" ::: "memory"); }

// TMA-staged variant of attn_prompt_kernel (the default when the pool has its 64-row tensor map):
// each 64-token K / V tile is DH/64 bulk tensor loads of 64 x 64 boxes (128-byte swizzle, so the
// ldmatrix reads are conflict-free without padding) completing on the pair buffer's mbarrier,
// issued by one thread; the Q rows still stream with cp.async. Same MMAs, masking, online softmax
// and merges as attn_prompt_kernel.
template <int DH>
struct PromptTmaSmem {
    static constexpr int kTileElems = kTile * DH;  // DH/64 boxes of 64 rows x 64 elements
    alignas(1024) __nv_bfloat16 k[2][2][kTileElems];  // [pair buffer][parity]
    alignas(1024) __nv_bfloat16 v[2][2][kTileElems];
    __nv_bfloat16 q[64][DH + 8];
    uint64_t bar[2];
};

// byte offset of (row, 16-byte chunk c over d_head) in a 64-row tile of 64-element boxes
DS_DEVICE uint32_t swz64(int row, int c) {
    return uint32_t((c >> 3) * (kTile * 128) + row * 128 + (((c & 7) ^ (row & 7)) << 4));
}

template <int DH>
__global__ void __launch_bounds__(kPromptWarps * 32)
attn_prompt_tma_kernel(const __grid_constant__ CUtensorMap tmap_kv, const __nv_bfloat16* __restrict__ q,
                       int n_h, const int32_t* __restrict__ row_pos, const int32_t* __restrict__ row_page_off,
                       const int32_t* __restrict__ flat_pages, const int32_t* __restrict__ blocks, KvLayout kv,
                       int layer, int splits, int stride, __nv_bfloat16* __restrict__ o, float* __restrict__ ws,
                       int* __restrict__ counters) {
    pdl_launch_dependents();
    extern __shared__ __align__(1024) uint8_t attn_smem_raw[];
    PromptTmaSmem<DH>& sm = *reinterpret_cast<PromptTmaSmem<DH>*>(
        (reinterpret_cast<uintptr_t>(attn_smem_raw) + 1023) & ~uintptr_t(1023));
    if (threadIdx.x == 0) {
        tma_prefetch_desc(&tmap_kv);
        mbar_init(&sm.bar[0], 1);
        mbar_init(&sm.bar[1], 1);
        fence_mbar_init();
    }
    __syncthreads();
    pdl_wait();
    constexpr int NT = DH / 8;
    constexpr int KS = DH / 16;
    constexpr int SN = kTile / 8;
    const int n_kv = kv.n_kv;
    const int G = n_h / n_kv;
    const int split = blockIdx.x % splits;
    const int kvh = (blockIdx.x / splits) % n_kv;
    const int bi = blockIdx.x / (splits * n_kv);
    const int t0 = blocks[3 * bi], npos = blocks[3 * bi + 1];
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int rg = warp & 3, par = warp >> 2;
    const int g = lane >> 2, tq = lane & 3;
    const int rows = npos * G;
    const int pos0 = row_pos[t0];
    const int last_pos = pos0 + npos - 1;
    const int n_tiles = (last_pos + kTile) / kTile;
    const int tile0 = split * n_tiles / splits, tile1 = (split + 1) * n_tiles / splits;
    const int32_t* pages = flat_pages + row_page_off[t0];

    const int r_base = rg * 16;
    const bool warp_active = r_base < rows;
    uint32_t qa[KS][4];
    const float qs = rsqrtf(float(DH)) * 1.4426950408889634f;
    for (int i = threadIdx.x; i < rows * (DH / 8); i += blockDim.x) {
        const int r = i / (DH / 8), c = (i % (DH / 8)) * 8;
        cp_async16(&sm.q[r][c], q + (size_t(t0 + r / G) * n_h + kvh * G + r % G) * DH + c);
    }
    cp_async_commit();
    int rpos[2];
#pragma unroll
    for (int hr = 0; hr < 2; ++hr) {
        const int r = r_base + g + 8 * hr;
        rpos[hr] = r < rows ? pos0 + r / G : -1;
    }
    float m_run[2] = {-INFINITY, -INFINITY}, l_run[2] = {0.f, 0.f};
    float acc[NT][4];
#pragma unroll
    for (int j = 0; j < NT; ++j) acc[j][0] = acc[j][1] = acc[j][2] = acc[j][3] = 0.f;

    const int row_k = (layer * 2 + 0) * n_kv + kvh;
    const int row_v = (layer * 2 + 1) * n_kv + kvh;
    const int rows_per_page = kv.n_layers * 2 * n_kv * 256;
    const int n_pairs = (tile1 - tile0 + 1) / 2;
    auto load_pair = [&](int pi, int buf) {  // thread 0 only
        const int nt_here = min(2, tile1 - (tile0 + 2 * pi));
        fence_proxy_async_smem();
        mbar_arrive_expect_tx(&sm.bar[buf], uint32_t(nt_here * 2 * kTile * DH * 2));
        for (int pp = 0; pp < nt_here; ++pp) {
            const int tok0 = (tile0 + 2 * pi + pp) * kTile;
            const int base = pages[tok0 >> 8] * rows_per_page + (tok0 & 255);
#pragma unroll
            for (int bx = 0; bx < DH / 64; ++bx) {
                tma_load_2d(&sm.k[buf][pp][bx * kTile * 64], &tmap_kv, &sm.bar[buf], bx * 64, base + row_k * 256);
                tma_load_2d(&sm.v[buf][pp][bx * kTile * 64], &tmap_kv, &sm.bar[buf], bx * 64, base + row_v * 256);
            }
        }
    };
    if (threadIdx.x == 0 && n_pairs > 0) load_pair(0, 0);
    cp_async_wait<0>();
    __syncthreads();
    if (warp_active) {  // Q fragments
#pragma unroll
        for (int kk = 0; kk < KS; ++kk)
            ldsm_x4(smem_u32(&sm.q[r_base + (lane & 15)][kk * 16 + (lane >> 4) * 8]), qa[kk][0], qa[kk][1],
                    qa[kk][2], qa[kk][3]);
    }
    for (int pi = 0; pi < n_pairs; ++pi) {
        const int buf = pi & 1;
        if (threadIdx.x == 0 && pi + 1 < n_pairs) load_pair(pi + 1, buf ^ 1);
        mbar_wait(&sm.bar[buf], uint32_t((pi >> 1) & 1));
        for (int pp = 0; pp < 2; ++pp) {  // zero V rows past the last valid token
            const int tile = tile0 + 2 * pi + pp;
            if (tile >= tile1) break;
            const int valid = min(kTile, last_pos + 1 - tile * kTile);
            uint8_t* vb = reinterpret_cast<uint8_t*>(&sm.v[buf][pp][0]);
            for (int i = threadIdx.x; i < (kTile - valid) * (DH / 8); i += blockDim.x) {
                const int r = valid + i / (DH / 8), c = i % (DH / 8);
                *reinterpret_cast<uint4*>(vb + swz64(r, c)) = make_uint4(0, 0, 0, 0);
            }
        }
        __syncthreads();
        const int tile = tile0 + 2 * pi + par;
        if (warp_active && tile < tile1) {
            const int tok0 = tile * kTile;
            float s[SN][4];
#pragma unroll
            for (int j = 0; j < SN; ++j) s[j][0] = s[j][1] = s[j][2] = s[j][3] = 0.f;
            const uint32_t kbase = smem_u32(&sm.k[buf][par][0]);
#pragma unroll
            for (int j = 0; j < SN; ++j)
#pragma unroll
                for (int kk = 0; kk < KS; kk += 2) {
                    const int mi = lane >> 3, rr = lane & 7;
                    uint32_t b0, b1, b2, b3;
                    ldsm_x4(kbase + swz64(j * 8 + rr, kk * 2 + mi), b0, b1, b2, b3);
                    mma16816(s[j], qa[kk], b0, b1);
                    mma16816(s[j], qa[kk + 1], b2, b3);
                }
            float mt[2] = {-INFINITY, -INFINITY};
#pragma unroll
            for (int j = 0; j < SN; ++j)
#pragma unroll
                for (int e = 0; e < 4; ++e) {
                    const int hr = e >> 1;
                    s[j][e] = tok0 + j * 8 + 2 * tq + (e & 1) > rpos[hr] ? -INFINITY : s[j][e] * qs;
                    mt[hr] = fmaxf(mt[hr], s[j][e]);
                }
            float alpha[2];
#pragma unroll
            for (int hr = 0; hr < 2; ++hr) {
                mt[hr] = fmaxf(mt[hr], __shfl_xor_sync(0xffffffffu, mt[hr], 1));
                mt[hr] = fmaxf(mt[hr], __shfl_xor_sync(0xffffffffu, mt[hr], 2));
                const float mn = fmaxf(m_run[hr], mt[hr]);
                alpha[hr] = mn == -INFINITY ? 1.f : exp2f(m_run[hr] - mn);
                m_run[hr] = mn;
            }
            float ls[2] = {0.f, 0.f};
            uint32_t pa[SN / 2][4];
#pragma unroll
            for (int j = 0; j < SN; ++j)
#pragma unroll
                for (int e = 0; e < 4; ++e) {
                    const int hr = e >> 1;
                    const float pv = m_run[hr] == -INFINITY ? 0.f : exp2f(s[j][e] - m_run[hr]);
                    s[j][e] = pv;
                    ls[hr] += pv;
                }
#pragma unroll
            for (int hr = 0; hr < 2; ++hr) l_run[hr] = l_run[hr] * alpha[hr] + ls[hr];
#pragma unroll
            for (int j = 0; j < NT; ++j) {
                acc[j][0] *= alpha[0];
                acc[j][1] *= alpha[0];
                acc[j][2] *= alpha[1];
                acc[j][3] *= alpha[1];
            }
#pragma unroll
            for (int kk = 0; kk < SN / 2; ++kk) {
                pa[kk][0] = pack2(s[2 * kk][0], s[2 * kk][1]);
                pa[kk][1] = pack2(s[2 * kk][2], s[2 * kk][3]);
                pa[kk][2] = pack2(s[2 * kk + 1][0], s[2 * kk + 1][1]);
                pa[kk][3] = pack2(s[2 * kk + 1][2], s[2 * kk + 1][3]);
            }
            const uint32_t vbase = smem_u32(&sm.v[buf][par][0]);
#pragma unroll
            for (int kk = 0; kk < SN / 2; ++kk)
#pragma unroll
                for (int nt = 0; nt < NT; nt += 2) {
                    const int mi = lane >> 3, rr = lane & 7;
                    uint32_t b0, b1, b2, b3;
                    ldsm_x4_t(vbase + swz64(kk * 16 + (mi & 1) * 8 + rr, nt + (mi >> 1)), b0, b1, b2, b3);
                    mma16816(acc[nt], pa[kk], b0, b1);
                    mma16816(acc[nt + 1], pa[kk], b2, b3);
                }
        }
        __syncthreads();  // pair buffer `buf` is refilled by the load of pair pi + 2
    }
#pragma unroll
    for (int hr = 0; hr < 2; ++hr) {
        l_run[hr] += __shfl_xor_sync(0xffffffffu, l_run[hr], 1);
        l_run[hr] += __shfl_xor_sync(0xffffffffu, l_run[hr], 2);
    }
    float* red = reinterpret_cast<float*>(&sm.k[0][0][0]);  // [4 row groups][16 rows][DH + 2]
    if (par == 1 && warp_active) {
#pragma unroll
        for (int hr = 0; hr < 2; ++hr) {
            float* dst = red + (rg * 16 + g + 8 * hr) * (DH + 2);
#pragma unroll
            for (int nt = 0; nt < NT; ++nt) {
                dst[nt * 8 + 2 * tq] = acc[nt][2 * hr];
                dst[nt * 8 + 2 * tq + 1] = acc[nt][2 * hr + 1];
            }
            if (tq == 0) {
                dst[DH] = m_run[hr];
                dst[DH + 1] = l_run[hr];
            }
        }
    }
    __syncthreads();
    if (par == 0 && warp_active) {
#pragma unroll
        for (int hr = 0; hr < 2; ++hr) {
            const int r = r_base + g + 8 * hr;
            const float* oth = red + (rg * 16 + g + 8 * hr) * (DH + 2);
            const float m1 = oth[DH], l1 = oth[DH + 1];
            const float M = fmaxf(m_run[hr], m1);
            const float w0 = m_run[hr] == -INFINITY ? 0.f : exp2f(m_run[hr] - M);
            const float w1 = m1 == -INFINITY ? 0.f : exp2f(m1 - M);
            const float L = l_run[hr] * w0 + l1 * w1;
            if (r >= rows) continue;
            const int p = r / G, h = r % G;
            const size_t row_head = size_t(t0 + p) * n_h + kvh * G + h;
            if (splits == 1) {
                const float inv = 1.0f / L;
                __nv_bfloat16* dst = o + row_head * DH;
#pragma unroll
                for (int nt = 0; nt < NT; ++nt) {
                    const int c = nt * 8 + 2 * tq;
                    *reinterpret_cast<uint32_t*>(dst + c) =
                        pack2((acc[nt][2 * hr] * w0 + oth[c] * w1) * inv, (acc[nt][2 * hr + 1] * w0 + oth[c + 1] * w1) * inv);
                }
            } else {
                float* dst = ws + (row_head * stride + split) * (DH + 2);
#pragma unroll
                for (int nt = 0; nt < NT; ++nt) {
                    const int c = nt * 8 + 2 * tq;
                    __stcg(dst + c, acc[nt][2 * hr] * w0 + oth[c] * w1);
                    __stcg(dst + c + 1, acc[nt][2 * hr + 1] * w0 + oth[c + 1] * w1);
                }
                if (tq == 0) {
                    __stcg(dst + DH, M);
                    __stcg(dst + DH + 1, L);
                }
            }
        }
    }
    if (splits == 1) return;
    __threadfence();
    __syncthreads();
    __shared__ int last_cta;
    if (threadIdx.x == 0) {
        int* cnt = counters + size_t(bi) * n_kv + kvh;
        const int old = atomicAdd(cnt, 1);
        last_cta = old == splits - 1;
        if (last_cta) *cnt = 0;
    }
    __syncthreads();
    if (!last_cta) return;
    __threadfence();
    for (int i = threadIdx.x; i < rows * DH; i += blockDim.x) {
        const int r = i / DH, dd = i % DH;
        const size_t row_head = size_t(t0 + r / G) * n_h + kvh * G + r % G;
        const float* base = ws + row_head * stride * (DH + 2);
        float M = -INFINITY;
        for (int sp = 0; sp < splits; ++sp) M = fmaxf(M, __ldcg(base + sp * (DH + 2) + DH));
        float num = 0.f, den = 0.f;
        for (int sp = 0; sp < splits; ++sp) {
            const float ms = __ldcg(base + sp * (DH + 2) + DH);
            if (ms == -INFINITY) continue;
            const float w = exp2f(ms - M);
            num += __ldcg(base + sp * (DH + 2) + dd) * w;
            den += __ldcg(base + sp * (DH + 2) + DH + 1) * w;
        }
        o[row_head * DH + dd] = f2bf(num / den);
    }
}

// ------------------------------------------------------ prompt blocks, tcgen05 ----
// Chunked-prefill attention on 5th-generation tensor cores (d_head 128, G <= 8): one CTA per
// (query block of 128 rows = 128/G prompt positions x G heads, KV head), FlashAttention-style
// over the request's 64-token KV tiles:
//   S  = Q . K^T   tcgen05.mma M=128 N=64 K=128, Q read from TMEM (stored there once by the
//                  softmax threads), K a K-major SW128 tile from TMA; S in TMEM
//   P  = softmax   one thread per row (TMEM lane), online max / sum in the log2 domain, P rows
//                  (bf16 pairs) stored back into TMEM (tcgen05.st) as the next MMA's A operand
//   O += P . V     tcgen05.mma M=128 N=128 K=64 with P read from TMEM and V as an MN-major B
//                  operand (the page layout [token][d_head] loaded by TMA, no transpose), O in
//                  TMEM -- P never touches shared memory, whose bandwidth bounds this kernel
// The softmax is a latency chain per tile (TMEM load -> max -> exp2 -> pack -> shared store ->
// fence -> arrive), so the tiles are split by parity between two independent softmax groups
// (warps 4-7: even tiles, warps 8-11: odd tiles), each with its own S buffer, P buffer, O
// accumulator, running max and sum: two chains in flight keep the tensor pipe fed (the
// FlashAttention-4 ping-pong, here over KV tiles of one query tile so Q and every K/V tile are
// staged once). The two partial softmax states merge in the epilogue. Each group moves its
// reference max lazily (rescales O / l only when a row's max passes it by > 8 in log2 units).
// Warp roles: w0 TMA producer of Q and the K ring, w1 / w3 MMA issuers of the even / odd group
// (S_{j+2} issued as soon as S_j is read, ahead of PV_j), w2 TMEM allocator then V-ring
// producer, w4-11 softmax.
// TMEM columns: S even [0, 64), S odd [64, 128), O even [128, 256), O odd [256, 384), P even
// [384, 416), P odd [416, 448), Q [448, 512). Shared memory carries only the K and V rings: with
// Q in shared memory an M128 N64 S step read 6 KB per 32-cycle dispatch and the operand reads
// plus the TMA writes bounded the tensor pipe at about half its floor.
constexpr int kTcRows = 128;
// K/V ring depth: a tile's MMAs take ~0.3 us, a TMA round trip from L2 / HBM ~1 us, so the loads
// run 3 tiles ahead (2 stages left them exposed)
constexpr int kTcStages = 4;
struct PromptTcSmem {
    alignas(1024) __nv_bfloat16 k[kTcStages][2][kTile * 64];     // [stage][dim half][token][64]
    alignas(1024) __nv_bfloat16 v[kTcStages][2][kTile * 64];     // [stage][dim half][token][64]
    float m_x[2][kTcRows], l_x[2][kTcRows];                      // [group][row] epilogue merge
    // per group g (tile parity): s_full / s_free (S buffer g), p_full / p_free (P buffer g and
    // the group's PV into O_g)
    // K and V rings are separate: K_j frees when S_j completes (long before PV_j), so the K loads
    // run further ahead than a joint ring allows
    uint64_t k_full[kTcStages], k_empty[kTcStages], v_full[kTcStages], v_empty[kTcStages];
    uint64_t q_full, s_full[2], s_free[2], p_full[2], p_free[2];
    uint32_t tmem;
};

// 2^x on the SFU without the denormal fix-up exp2f carries (P underflow to 0 is harmless)
__device__ __forceinline__ float ex2_sfu(float x) {
    float y;
    asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
    return y;
}
__device__ __forceinline__ void sts128(uint32_t addr, uint32_t a, uint32_t b, uint32_t c, uint32_t d) {
    asm volatile("st.shared.v4.b32 [%0], {%1, %2, %3, %4};" ::"r"(addr), "r"(a), "r"(b), "r"(c), "r"(d)
                 : "memory");
}

template <int G>
__global__ void __launch_bounds__(384)
attn_prompt_tc_kernel(const __grid_constant__ CUtensorMap tmap_kv, const __nv_bfloat16* __restrict__ q,
                      int n_h, const int32_t* __restrict__ row_pos, const int32_t* __restrict__ row_page_off,
                      const int32_t* __restrict__ flat_pages, const int32_t* __restrict__ blocks, KvLayout kv,
                      int layer, __nv_bfloat16* __restrict__ o, int dbg) {
    constexpr int DH = 128;
    extern __shared__ __align__(1024) uint8_t tc_smem_raw[];
    PromptTcSmem& sm = *reinterpret_cast<PromptTcSmem*>(
        (reinterpret_cast<uintptr_t>(tc_smem_raw) + 1023) & ~uintptr_t(1023));
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int n_kv = kv.n_kv;
    const int kvh = blockIdx.x % n_kv;
    // blocks in reverse: a request's later query blocks walk more KV tiles, so the longest CTAs
    // start in the first wave and the short ones fill the tail
    const int bi = int(gridDim.x) / n_kv - 1 - int(blockIdx.x) / n_kv;
    if (threadIdx.x == 0) {
        tma_prefetch_desc(&tmap_kv);
        for (int b = 0; b < kTcStages; ++b) {
            mbar_init(&sm.k_full[b], 1);
            mbar_init(&sm.k_empty[b], 1);
            mbar_init(&sm.v_full[b], 1);
            mbar_init(&sm.v_empty[b], 1);
        }
        mbar_init(&sm.q_full, 256);
        for (int g = 0; g < 2; ++g) {
            mbar_init(&sm.s_full[g], 1);
            mbar_init(&sm.s_free[g], 128);
            mbar_init(&sm.p_full[g], 128);
            mbar_init(&sm.p_free[g], 1);
        }
        fence_mbar_init();
    }
    if (warp == 2) tmem_alloc(&sm.tmem, 512);
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    // dependents launch only once every CTA holds its TMEM: a PDL-launched GEMM CTA that took
    // columns first on this SM would wait for this grid while this CTA waits for its columns
    pdl_launch_dependents();
    const uint32_t tmem = sm.tmem;
    pdl_wait();
    const int t0 = blocks[3 * bi], npos = blocks[3 * bi + 1];
    const int rows = npos * G;
    const int pos0 = row_pos[t0];
    const int last_pos = pos0 + npos - 1;
    const int n_tiles = (last_pos + kTile) / kTile;
    const int32_t* pages = flat_pages + row_page_off[t0];
    const int rows_per_page = kv.n_layers * 2 * n_kv * 256;
    const int row_k = (layer * 2 + 0) * n_kv + kvh, row_v = (layer * 2 + 1) * n_kv + kvh;

    if (warp == 0) {
        if (lane == 0) {
            for (int j = 0; j < n_tiles; ++j) {  // K tiles
                const int st = j % kTcStages;
                if (j >= kTcStages) mbar_wait(&sm.k_empty[st], uint32_t((j / kTcStages - 1) & 1));
                const int tok0 = j * kTile;
                const int base = pages[tok0 >> 8] * rows_per_page + (tok0 & 255);
                if (dbg & 8) { mbar_arrive(&sm.k_full[st]); continue; }
                mbar_arrive_expect_tx(&sm.k_full[st], uint32_t(kTile * DH * 2));
                for (int bx = 0; bx < 2; ++bx)
                    tma_load_2d(&sm.k[st][bx][0], &tmap_kv, &sm.k_full[st], bx * 64, base + row_k * 256);
            }
        }
    } else if (warp == 2) {
        if (lane == 0) {
            for (int j = 0; j < n_tiles; ++j) {  // V tiles
                const int st = j % kTcStages;
                if (j >= kTcStages) mbar_wait(&sm.v_empty[st], uint32_t((j / kTcStages - 1) & 1));
                const int tok0 = j * kTile;
                const int base = pages[tok0 >> 8] * rows_per_page + (tok0 & 255);
                if (dbg & 8) { mbar_arrive(&sm.v_full[st]); continue; }
                mbar_arrive_expect_tx(&sm.v_full[st], uint32_t(kTile * DH * 2));
                for (int bx = 0; bx < 2; ++bx)
                    tma_load_2d(&sm.v[st][bx][0], &tmap_kv, &sm.v_full[st], bx * 64, base + row_v * 256);
            }
        }
    } else if (warp == 1 || warp == 3) {
        // one MMA issuer per softmax group (warp 1: even tiles, warp 3: odd tiles): with one
        // issuer for both groups, each group's S and PV issue waited behind the other group's
        // barriers (measured 180 -> 162 us on a 3840-token prompt with the split)
        {  // the whole warp runs the loop; one elected lane issues each MMA / commit
            const int g = warp >> 1;
            const uint32_t idesc_s = umma_idesc_bf16(kTcRows, kTile);
            const uint32_t idesc_o = umma_idesc_bf16_bmn(kTcRows, DH);
            auto issue_s = [&](int j) {  // S_j = Q . K_j^T into S buffer g
                const int st = j % kTcStages;
                mbar_wait(&sm.k_full[st], uint32_t((j / kTcStages) & 1));
                if (j >= 2) mbar_wait(&sm.s_free[g], uint32_t(((j >> 1) - 1) & 1));  // S_{j-2} read out
                tc_fence_after();
#pragma unroll
                for (int ks = 0; ks < DH / 16; ++ks) {
                    if (dbg & 4) break;
                    const uint32_t a = tmem + 448 + uint32_t(ks * 8);  // Q: 16 dims = 8 columns
                    const uint64_t b = umma_sdesc_sw128(smem_u32(&sm.k[st][ks >> 2][0]) + (ks & 3) * 32);
                    umma_bf16_ts_warp(tmem + uint32_t(g * kTile), a, b, idesc_s, ks > 0 ? 1u : 0u);
                }
                umma_commit_warp(&sm.s_full[g]);
                umma_commit_warp(&sm.k_empty[st]);
            };
            mbar_wait(&sm.q_full, 0);  // Q in TMEM
            if (g < n_tiles) issue_s(g);
            for (int j = g; j < n_tiles; j += 2) {
                const int st = j % kTcStages;
                // S_{j+2} as soon as the group has read S_j, ahead of PV_j
                if (j + 2 < n_tiles) issue_s(j + 2);
                mbar_wait(&sm.p_full[g], uint32_t((j >> 1) & 1));  // P_j written, O_g rescaled
                mbar_wait(&sm.v_full[st], uint32_t((j / kTcStages) & 1));
                tc_fence_after();
#pragma unroll
                for (int ks = 0; ks < kTile / 16; ++ks) {  // O_g += P_j . V_j
                    if (dbg & 2) break;
                    // P: 16 tokens per step = 8 TMEM columns of bf16 pairs
                    const uint32_t a = tmem + 384 + uint32_t(g * (kTile / 2) + ks * 8);
                    // V: 16 tokens per step = two 8-token groups of 1024 B; dim halves 8 KB apart
                    const uint64_t b = umma_sdesc_sw128_mn(smem_u32(&sm.v[st][0][0]) + ks * 2048, 8192, 1024);
                    umma_bf16_ts_warp(tmem + 128 + uint32_t(g * DH), a, b, idesc_o, (j >= 2 || ks > 0) ? 1u : 0u);
                }
                umma_commit_warp(&sm.p_free[g]);
                umma_commit_warp(&sm.v_empty[st]);
            }
        }
    } else if (warp >= 4) {
        const int grp = (warp - 4) >> 2, quarter = warp & 3;
        const int r = quarter * 32 + lane;  // this thread's row = TMEM lane
        const uint32_t lane_off = uint32_t(quarter * 32) << 16;
        const uint32_t o_col = 128 + uint32_t(grp * DH);
        const int my_pos = r < rows ? pos0 + r / G : -1;
        const float qs = rsqrtf(float(DH)) * 1.4426950408889634f;
        const uint32_t p_col = 384 + uint32_t(grp * (kTile / 2));
        {  // Q row r, dims [64 grp, 64 grp + 64), into TMEM columns 448 + 32 grp (bf16 pairs)
            uint32_t qv[32];
            if (r < rows) {
                const uint4* src = reinterpret_cast<const uint4*>(
                    q + (size_t(t0 + r / G) * n_h + kvh * G + r % G) * DH + grp * 64);
#pragma unroll
                for (int c = 0; c < 8; ++c) {
                    const uint4 v4 = __ldg(src + c);
                    qv[4 * c] = v4.x, qv[4 * c + 1] = v4.y, qv[4 * c + 2] = v4.z, qv[4 * c + 3] = v4.w;
                }
            } else {
#pragma unroll
                for (int c = 0; c < 32; ++c) qv[c] = 0u;
            }
            tmem_st16(tmem + lane_off + 448 + uint32_t(grp * 32), qv);
            tmem_st16(tmem + lane_off + 448 + uint32_t(grp * 32 + 16), qv + 16);
            tmem_st_wait();
            tc_fence_before();
            mbar_arrive(&sm.q_full);
        }
        float m_ref = -INFINITY, l_run = 0.f;
        for (int j = grp; j < n_tiles; j += 2) {
            const int st = j % kTcStages, u = j >> 1;  // u: this group's use count of its buffers
            const int tok0 = j * kTile;
            mbar_wait(&sm.s_full[grp], uint32_t(u & 1));
            tc_fence_after();
            float sv[kTile];
#pragma unroll
            for (int c = 0; c < kTile; c += 16)
                tmem_ld16(tmem + lane_off + uint32_t(grp * kTile + c), reinterpret_cast<uint32_t*>(sv + c));
            tmem_ld_wait();
            tc_fence_before();
            mbar_arrive(&sm.s_free[grp]);
            // max over the raw scores (the scale qs > 0 keeps the order), scaled once; the causal
            // mask only touches the tiles that reach this row's position
            if (tok0 + kTile - 1 > my_pos) {
#pragma unroll
                for (int c = 0; c < kTile; ++c)
                    if (tok0 + c > my_pos) sv[c] = -INFINITY;
            }
            float mt = -INFINITY;
#pragma unroll
            for (int c = 0; c < kTile; ++c) mt = fmaxf(mt, sv[c]);
            mt *= qs;
            const bool move = mt > m_ref + 8.0f;  // includes the first finite max (m_ref = -inf)
            const float m_new = move ? mt : m_ref;
            const float alpha = (!move || m_ref == -INFINITY) ? 1.f : ex2_sfu(m_ref - m_new);
            m_ref = m_new;
            const float neg_m = m_new == -INFINITY ? 0.f : -m_new;  // all-masked row: exp2(-inf) = 0
            float ls = 0.f;
            uint32_t pk[kTile / 2];
#pragma unroll
            for (int c = 0; c < kTile; c += 2) {
                const float p0 = (dbg & 1) ? sv[c] : ex2_sfu(fmaf(sv[c], qs, neg_m));
                const float p1 = (dbg & 1) ? sv[c + 1] : ex2_sfu(fmaf(sv[c + 1], qs, neg_m));
                ls += p0 + p1;
                pk[c / 2] = pack2(p0, p1);
            }
            l_run = l_run * alpha + ls;
            // this group's previous PV (tile j-2) done: O_g stable and P buffer g free. The
            // window is exact: the group awaited the use before it at tile j-2.
            if (j >= 2) {
                mbar_wait(&sm.p_free[grp], uint32_t((u - 1) & 1));
                tc_fence_after();
                if (__any_sync(0xffffffffu, alpha != 1.f)) {
#pragma unroll
                    for (int c = 0; c < DH; c += 16) {
                        uint32_t ov[16];
                        tmem_ld16(tmem + lane_off + o_col + uint32_t(c), ov);
                        tmem_ld_wait();
#pragma unroll
                        for (int e = 0; e < 16; ++e) ov[e] = __float_as_uint(__uint_as_float(ov[e]) * alpha);
                        tmem_st16(tmem + lane_off + o_col + uint32_t(c), ov);
                    }
                    tmem_st_wait();
                }
            }
            // P row r: 32 columns of bf16 pairs in this lane
            tmem_st16(tmem + lane_off + p_col, pk);
            tmem_st16(tmem + lane_off + p_col + 16, pk + 16);
            // V rows past the last valid token must be zero (0 * garbage must not be NaN)
            const int valid = min(kTile, last_pos + 1 - tok0);
            if (valid < kTile) {
                mbar_wait(&sm.v_full[st], uint32_t((j / kTcStages) & 1));  // V_j landed
                for (int i = r; i < (kTile - valid) * 16; i += 128) {
                    const int tr = valid + i / 16, c = i % 16;  // token row, 16-byte chunk over 128 dims
                    sts128(smem_u32(&sm.v[st][c >> 3][0]) + uint32_t(tr * 128 + (((c & 7) ^ (tr & 7)) << 4)), 0, 0, 0, 0);
                }
                fence_proxy_async_smem();  // the zeroed V rows are read by the MMA's async proxy
            }
            tmem_st_wait();
            tc_fence_before();
            mbar_arrive(&sm.p_full[grp]);
        }
        // epilogue: merge the two groups' (O, max, sum) per row; group g writes O columns
        // [64 g, 64 g + 64). The exchange comes first: after it the partner has passed its own
        // last P-buffer wait, so both groups' final PV waits below have exact parity windows.
        sm.m_x[grp][r] = m_ref;
        sm.l_x[grp][r] = l_run;
        asm volatile("bar.sync %0, 64;" ::"r"(1 + quarter) : "memory");  // warps w and w + 4
        const float m0 = sm.m_x[0][r], m1 = sm.m_x[1][r];
        const float mx = fmaxf(m0, m1);
        const float a0 = m0 == -INFINITY ? 0.f : ex2_sfu(m0 - mx);
        const float a1 = m1 == -INFINITY ? 0.f : ex2_sfu(m1 - mx);
        const float l_row = sm.l_x[0][r] * a0 + sm.l_x[1][r] * a1;
        const int n_g[2] = {(n_tiles + 1) >> 1, n_tiles >> 1};  // tiles per group
#pragma unroll
        for (int g = 0; g < 2; ++g)
            if (n_g[g] > 0) mbar_wait(&sm.p_free[g], uint32_t((n_g[g] - 1) & 1));
        tc_fence_after();
        const float inv = l_row > 0.f ? 1.0f / l_row : 0.f;
        const float w0 = a0 * inv, w1 = n_g[1] > 0 ? a1 * inv : 0.f;
        __nv_bfloat16* dst =
            r < rows ? o + (size_t(t0 + r / G) * n_h + kvh * G + r % G) * DH + grp * (DH / 2) : nullptr;
#pragma unroll
        for (int c = 0; c < DH / 2; c += 16) {
            const uint32_t col = uint32_t(grp * (DH / 2) + c);
            uint32_t o0[16], o1[16];
            tmem_ld16(tmem + lane_off + 128 + col, o0);
            if (n_g[1] > 0) tmem_ld16(tmem + lane_off + 128 + DH + col, o1);
            tmem_ld_wait();
            if (dst) {
                float f[16];
#pragma unroll
                for (int e = 0; e < 16; ++e)
                    f[e] = __uint_as_float(o0[e]) * w0 + (n_g[1] > 0 ? __uint_as_float(o1[e]) * w1 : 0.f);
                reinterpret_cast<uint4*>(dst + c)[0] = pack8(f);
                reinterpret_cast<uint4*>(dst + c)[1] = pack8(f + 8);
            }
        }
    }
    tc_fence_before();
    __syncthreads();
    if (warp == 2) {
        tc_fence_after();
        tmem_dealloc(tmem, 512);
    }
}

// ------------------------------------------------------------------ decode rows ----
// One decode row x one KV head x one context split per CTA. The split's context is cut into
// 16-token chunks dealt round-robin to the 4 warps; every warp streams its chunks through its
// own ST-deep cp.async ring (no CTA-wide barrier in the loop), computes S = Q.K^T and
// O += P.V with mma.sync (the G <= 16 query heads of the KV head are the M rows), and the 4
// partial softmax states merge through shared memory at the end. Memory-level parallelism:
// (ST - 1) x 8 KB of K/V in flight per warp while it computes on the previous chunk.
constexpr int kDecChunk = 16;
constexpr int kDecStages = 2;  // per-warp ring depth; 2 keeps 3 CTAs (12 warps) resident per SM

template <int DH, int ST = kDecStages>
struct DecSmem {
    __nv_bfloat16 k[kAttnWarps][ST][kDecChunk][DH + 8];
    __nv_bfloat16 v[kAttnWarps][ST][kDecChunk][DH + 8];
};

template <int DH, int ST = kDecStages>
__global__ void __launch_bounds__(kAttnWarps * 32)
attn_decode_kernel(const __nv_bfloat16* __restrict__ q, int n_h, const int32_t* __restrict__ row_pos,
                   const int32_t* __restrict__ row_page_off, const int32_t* __restrict__ flat_pages,
                   const int32_t* __restrict__ drows, KvLayout kv, int layer, int splits, int stride,
                   __nv_bfloat16* __restrict__ o, float* __restrict__ ws, int* __restrict__ counters,
                   L2Prefetch pf) {
    pdl_launch_dependents();
    l2_prefetch_slice(pf);
    pdl_wait();
    extern __shared__ __align__(16) uint8_t dec_smem[];
    DecSmem<DH, ST>& sm = *reinterpret_cast<DecSmem<DH, ST>*>(dec_smem);
    constexpr int NT = DH / 8, KS = DH / 16;
    const int n_kv = kv.n_kv;
    const int G = n_h / n_kv;
    const int split = blockIdx.x % splits;
    const int kvh = (blockIdx.x / splits) % n_kv;
    const int t = drows[blockIdx.x / (splits * n_kv)];
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int g = lane >> 2, tq = lane & 3;
    const int ctx = row_pos[t] + 1;
    const int n_chunks = (ctx + kDecChunk - 1) / kDecChunk;
    const int ch0 = split * n_chunks / splits, ch1 = (split + 1) * n_chunks / splits;
    const int32_t* pages = flat_pages + row_page_off[t];

    uint32_t qa[KS][4];
    const float qs = rsqrtf(float(DH)) * 1.4426950408889634f;
#pragma unroll
    for (int kk = 0; kk < KS; ++kk)
#pragma unroll
        for (int i = 0; i < 4; ++i) {
            const int r = g + ((i & 1) ? 8 : 0);
            const int col = kk * 16 + 2 * tq + ((i & 2) ? 8 : 0);
            float x0 = 0.f, x1 = 0.f;
            if (r < G) {
                const __nv_bfloat162 v2 = *reinterpret_cast<const __nv_bfloat162*>(
                    q + (size_t(t) * n_h + kvh * G + r) * DH + col);
                x0 = __bfloat162float(v2.x) * qs;
                x1 = __bfloat162float(v2.y) * qs;
            }
            qa[kk][i] = pack2(x0, x1);
        }
    float m_run[2] = {-INFINITY, -INFINITY}, l_run[2] = {0.f, 0.f};
    float acc[NT][4];
#pragma unroll
    for (int j = 0; j < NT; ++j) acc[j][0] = acc[j][1] = acc[j][2] = acc[j][3] = 0.f;

    const size_t head_k = ((size_t(layer) * 2 + 0) * n_kv + kvh) * 256 * DH;
    const size_t head_v = ((size_t(layer) * 2 + 1) * n_kv + kvh) * 256 * DH;
    // this warp's chunks: ch0 + warp, ch0 + warp + 4, ...
    const int my_n = ch1 - ch0 > warp ? (ch1 - ch0 - warp + kAttnWarps - 1) / kAttnWarps : 0;
    auto load = [&](int j, int buf) {
        const int tok0 = (ch0 + warp + j * kAttnWarps) * kDecChunk;
        const size_t base = size_t(pages[tok0 >> 8]) * kv.page_elems + size_t(tok0 & 255) * DH;
        const __nv_bfloat16* ksrc = kv.pool + base + head_k;
        const __nv_bfloat16* vsrc = kv.pool + base + head_v;
#pragma unroll
        for (int i = lane; i < kDecChunk * DH / 8; i += 32) {
            const int r = i / (DH / 8), c = (i % (DH / 8)) * 8;
            cp_async16(&sm.k[warp][buf][r][c], ksrc + size_t(r) * DH + c);
            cp_async16(&sm.v[warp][buf][r][c], vsrc + size_t(r) * DH + c);
        }
    };
#pragma unroll
    for (int j = 0; j < ST - 1; ++j) {
        if (j < my_n) load(j, j);
        cp_async_commit();
    }
    for (int j = 0; j < my_n; ++j) {
        const int buf = j % ST;
        // refill the slot chunk j-1 used (consumed: __syncwarp at the end of the last iteration)
        if (j + ST - 1 < my_n) load(j + ST - 1, (j + ST - 1) % ST);
        cp_async_commit();
        cp_async_wait<ST - 1>();
        __syncwarp();
        const int tok0 = (ch0 + warp + j * kAttnWarps) * kDecChunk;
        const int valid = min(kDecChunk, ctx - tok0);
        if (valid < kDecChunk) {  // no 0 * garbage = NaN from rows past the context
            for (int i = lane; i < (kDecChunk - valid) * (DH / 8); i += 32) {
                const int r = valid + i / (DH / 8), c = (i % (DH / 8)) * 8;
                *reinterpret_cast<uint4*>(&sm.v[warp][buf][r][c]) = make_uint4(0, 0, 0, 0);
            }
            __syncwarp();
        }
        float s[2][4];
#pragma unroll
        for (int jn = 0; jn < 2; ++jn) {
            s[jn][0] = s[jn][1] = s[jn][2] = s[jn][3] = 0.f;
            const uint32_t kbase = smem_u32(&sm.k[warp][buf][0][0]);
#pragma unroll
            for (int kk = 0; kk < KS; kk += 2) {
                const int mi = lane >> 3, rr = lane & 7;
                uint32_t b0, b1, b2, b3;
                ldsm_x4(kbase + uint32_t(((jn * 8 + rr) * (DH + 8) + kk * 16 + mi * 8) * 2), b0, b1, b2, b3);
                mma16816(s[jn], qa[kk], b0, b1);
                mma16816(s[jn], qa[kk + 1], b2, b3);
            }
        }
        float mt[2] = {-INFINITY, -INFINITY};
#pragma unroll
        for (int jn = 0; jn < 2; ++jn)
#pragma unroll
            for (int e = 0; e < 4; ++e) {
                const int tok = tok0 + jn * 8 + 2 * tq + (e & 1);
                if (tok >= ctx) s[jn][e] = -INFINITY;
                mt[e >> 1] = fmaxf(mt[e >> 1], s[jn][e]);
            }
        float alpha[2];
#pragma unroll
        for (int hr = 0; hr < 2; ++hr) {
            mt[hr] = fmaxf(mt[hr], __shfl_xor_sync(0xffffffffu, mt[hr], 1));
            mt[hr] = fmaxf(mt[hr], __shfl_xor_sync(0xffffffffu, mt[hr], 2));
            const float mn = fmaxf(m_run[hr], mt[hr]);
            alpha[hr] = mn == -INFINITY ? 1.f : exp2f(m_run[hr] - mn);
            m_run[hr] = mn;
        }
#pragma unroll
        for (int jn = 0; jn < 2; ++jn)
#pragma unroll
            for (int e = 0; e < 4; ++e) {
                const int hr = e >> 1;
                s[jn][e] = m_run[hr] == -INFINITY ? 0.f : exp2f(s[jn][e] - m_run[hr]);
            }
        float ls[2];
        ls[0] = s[0][0] + s[0][1] + s[1][0] + s[1][1];
        ls[1] = s[0][2] + s[0][3] + s[1][2] + s[1][3];
        l_run[0] = l_run[0] * alpha[0] + ls[0];
        l_run[1] = l_run[1] * alpha[1] + ls[1];
        // the running max rarely moves after the first chunks: skip the 64-FMUL rescale then
        if (__any_sync(0xffffffffu, alpha[0] != 1.f || alpha[1] != 1.f)) {
#pragma unroll
            for (int nt = 0; nt < NT; ++nt) {
                acc[nt][0] *= alpha[0];
                acc[nt][1] *= alpha[0];
                acc[nt][2] *= alpha[1];
                acc[nt][3] *= alpha[1];
            }
        }
        uint32_t pa[4] = {pack2(s[0][0], s[0][1]), pack2(s[0][2], s[0][3]), pack2(s[1][0], s[1][1]),
                          pack2(s[1][2], s[1][3])};
        const uint32_t vbase = smem_u32(&sm.v[warp][buf][0][0]);
#pragma unroll
        for (int nt = 0; nt < NT; nt += 2) {
            const int mi = lane >> 3, rr = lane & 7;
            uint32_t b0, b1, b2, b3;
            ldsm_x4_t(vbase + uint32_t((((mi & 1) * 8 + rr) * (DH + 8) + (nt + (mi >> 1)) * 8) * 2), b0, b1,
                      b2, b3);
            mma16816(acc[nt], pa, b0, b1);
            mma16816(acc[nt + 1], pa, b2, b3);
        }
        __syncwarp();
    }
    cp_async_wait<0>();
#pragma unroll
    for (int hr = 0; hr < 2; ++hr) {
        l_run[hr] += __shfl_xor_sync(0xffffffffu, l_run[hr], 1);
        l_run[hr] += __shfl_xor_sync(0xffffffffu, l_run[hr], 2);
    }
    // merge the 4 warps' states through shared memory (reusing the K ring)
    __syncthreads();
    float* red = reinterpret_cast<float*>(&sm.k[0][0][0][0]);  // [4 warps][16 rows][DH + 2]
#pragma unroll
    for (int hr = 0; hr < 2; ++hr) {
        const int r = g + 8 * hr;
        float* dst = red + (warp * 16 + r) * (DH + 2);
#pragma unroll
        for (int nt = 0; nt < NT; ++nt) {
            dst[nt * 8 + 2 * tq] = acc[nt][2 * hr];
            dst[nt * 8 + 2 * tq + 1] = acc[nt][2 * hr + 1];
        }
        if (tq == 0) {
            dst[DH] = m_run[hr];
            dst[DH + 1] = l_run[hr];
        }
    }
    __syncthreads();
    for (int i = threadIdx.x; i < G * DH; i += blockDim.x) {
        const int r = i / DH, dd = i % DH;
        float M = -INFINITY;
#pragma unroll
        for (int w = 0; w < kAttnWarps; ++w) M = fmaxf(M, red[(w * 16 + r) * (DH + 2) + DH]);
        float num = 0.f, den = 0.f;
#pragma unroll
        for (int w = 0; w < kAttnWarps; ++w) {
            const float* src = red + (w * 16 + r) * (DH + 2);
            const float wt = src[DH] == -INFINITY ? 0.f : exp2f(src[DH] - M);
            num += src[dd] * wt;
            den += src[DH + 1] * wt;
        }
        const size_t row_head = size_t(t) * n_h + kvh * G + r;
        if (splits == 1) {
            o[row_head * DH + dd] = f2bf(num / den);
        } else {
            float* dst = ws + (row_head * stride + split) * (DH + 2);
            __stcg(dst + dd, num);
            if (dd == 0) {
                __stcg(dst + DH, M);
                __stcg(dst + DH + 1, den);
            }
        }
    }
    if (splits == 1) return;
    // context splits: the last CTA of this (row, KV head) to finish merges every split's partial
    // in split order (deterministic) -- no separate combine launch
    __threadfence();
    __syncthreads();
    __shared__ int last_cta;
    if (threadIdx.x == 0) {
        int* cnt = counters + size_t(t) * n_kv + kvh;
        const int old = atomicAdd(cnt, 1);
        last_cta = old == splits - 1;
        if (last_cta) *cnt = 0;  // ready for the next launch
    }
    __syncthreads();
    if (!last_cta) return;
    __threadfence();
    for (int i = threadIdx.x; i < G * DH; i += blockDim.x) {
        const int r = i / DH, dd = i % DH;
        const size_t row_head = size_t(t) * n_h + kvh * G + r;
        const float* base = ws + row_head * stride * (DH + 2);
        float M = -INFINITY;
        for (int sp = 0; sp < splits; ++sp) M = fmaxf(M, __ldcg(base + sp * (DH + 2) + DH));
        float num = 0.f, den = 0.f;
        for (int sp = 0; sp < splits; ++sp) {
            const float ms = __ldcg(base + sp * (DH + 2) + DH);
            if (ms == -INFINITY) continue;
            const float w = exp2f(ms - M);
            num += __ldcg(base + sp * (DH + 2) + dd) * w;
            den += __ldcg(base + sp * (DH + 2) + DH + 1) * w;
        }
        o[row_head * DH + dd] = f2bf(num / den);
    }
}

DS_DEVICE uint32_t movmatrix_t(uint32_t a) {
    uint32_t d;
    asm volatile("movmatrix.sync.aligned.m8n8.trans.b16 %0, %1;" : "=r"(d) : "r"(a));
    return d;
}

// Operand-swapped decode rows (G <= 8 query heads per KV head): S^T = K . Q^T with the 16 chunk
// tokens as the MMA M rows and the heads as N (8 columns, G real) and O^T += V^T . P^T with
// 16 head dims as M -- half the mma.sync and softmax work of the Q-as-M form (where only G of
// the 16 M rows are real), fewer accumulator registers. P^T moves from the accumulator layout
// into the B-operand layout with movmatrix. Same ring / split / merge structure as
// attn_decode_kernel.
template <int DH, int ST = kDecStages>
__global__ void __launch_bounds__(kAttnWarps * 32)
attn_decode_t_kernel(const __nv_bfloat16* __restrict__ q, int n_h, const int32_t* __restrict__ row_pos,
                     const int32_t* __restrict__ row_page_off, const int32_t* __restrict__ flat_pages,
                     const int32_t* __restrict__ drows, KvLayout kv, int layer, int splits, int stride,
                     __nv_bfloat16* __restrict__ o, float* __restrict__ ws, int* __restrict__ counters,
                     L2Prefetch pf) {
    pdl_launch_dependents();
    l2_prefetch_slice(pf);
    pdl_wait();
    extern __shared__ __align__(16) uint8_t dec_smem[];
    DecSmem<DH, ST>& sm = *reinterpret_cast<DecSmem<DH, ST>*>(dec_smem);
    constexpr int KS = DH / 16;  // k-steps of S^T and M tiles of O^T
    const int n_kv = kv.n_kv;
    const int G = n_h / n_kv;
    const int split = blockIdx.x % splits;
    const int kvh = (blockIdx.x / splits) % n_kv;
    const int t = drows[blockIdx.x / (splits * n_kv)];
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int g = lane >> 2, tq = lane & 3;
    const int ctx = row_pos[t] + 1;
    const int n_chunks = (ctx + kDecChunk - 1) / kDecChunk;
    const int ch0 = split * n_chunks / splits, ch1 = (split + 1) * n_chunks / splits;
    const int32_t* pages = flat_pages + row_page_off[t];

    // Q^T as the B operand (k = head dim, n = head g): b0 = dims 2tq..+1, b1 = dims 2tq+8..+9
    uint32_t qb[KS][2];
    const float qs = rsqrtf(float(DH)) * 1.4426950408889634f;
#pragma unroll
    for (int kk = 0; kk < KS; ++kk)
#pragma unroll
        for (int i = 0; i < 2; ++i) {
            float x0 = 0.f, x1 = 0.f;
            if (g < G) {
                const __nv_bfloat162 v2 = *reinterpret_cast<const __nv_bfloat162*>(
                    q + (size_t(t) * n_h + kvh * G + g) * DH + kk * 16 + 2 * tq + 8 * i);
                x0 = __bfloat162float(v2.x) * qs;
                x1 = __bfloat162float(v2.y) * qs;
            }
            qb[kk][i] = pack2(x0, x1);
        }
    // per head column (2tq, 2tq+1): running max and this thread's partial row sum
    float m_run[2] = {-INFINITY, -INFINITY}, l_run[2] = {0.f, 0.f};
    float acc[KS][4];  // O^T tile mt: dims mt*16 + g (+8), heads 2tq, 2tq+1
#pragma unroll
    for (int j = 0; j < KS; ++j) acc[j][0] = acc[j][1] = acc[j][2] = acc[j][3] = 0.f;

    const size_t head_k = ((size_t(layer) * 2 + 0) * n_kv + kvh) * 256 * DH;
    const size_t head_v = ((size_t(layer) * 2 + 1) * n_kv + kvh) * 256 * DH;
    const int my_n = ch1 - ch0 > warp ? (ch1 - ch0 - warp + kAttnWarps - 1) / kAttnWarps : 0;
    auto load = [&](int j, int buf) {
        const int tok0 = (ch0 + warp + j * kAttnWarps) * kDecChunk;
        const size_t base = size_t(pages[tok0 >> 8]) * kv.page_elems + size_t(tok0 & 255) * DH;
        const __nv_bfloat16* ksrc = kv.pool + base + head_k;
        const __nv_bfloat16* vsrc = kv.pool + base + head_v;
#pragma unroll
        for (int i = lane; i < kDecChunk * DH / 8; i += 32) {
            const int r = i / (DH / 8), c = (i % (DH / 8)) * 8;
            cp_async16(&sm.k[warp][buf][r][c], ksrc + size_t(r) * DH + c);
            cp_async16(&sm.v[warp][buf][r][c], vsrc + size_t(r) * DH + c);
        }
    };
#pragma unroll
    for (int j = 0; j < ST - 1; ++j) {
        if (j < my_n) load(j, j);
        cp_async_commit();
    }
    for (int j = 0; j < my_n; ++j) {
        const int buf = j % ST;
        if (j + ST - 1 < my_n) load(j + ST - 1, (j + ST - 1) % ST);
        cp_async_commit();
        cp_async_wait<ST - 1>();
        __syncwarp();
        const int tok0 = (ch0 + warp + j * kAttnWarps) * kDecChunk;
        const int valid = min(kDecChunk, ctx - tok0);
        if (valid < kDecChunk) {  // no 0 * garbage = NaN from rows past the context
            for (int i = lane; i < (kDecChunk - valid) * (DH / 8); i += 32) {
                const int r = valid + i / (DH / 8), c = (i % (DH / 8)) * 8;
                *reinterpret_cast<uint4*>(&sm.v[warp][buf][r][c]) = make_uint4(0, 0, 0, 0);
            }
            __syncwarp();
        }
        // S^T[16 tokens][8 heads]
        float s[4] = {0.f, 0.f, 0.f, 0.f};
        const uint32_t kbase = smem_u32(&sm.k[warp][buf][0][0]);
#pragma unroll
        for (int kk = 0; kk < KS; ++kk) {
            uint32_t a[4];
            // A = K rows (tokens) x 16 dims: lanes 0-15 rows 0-15 at col kk*16, lanes 16-31 at +8
            ldsm_x4(kbase + uint32_t(((lane & 15) * (DH + 8) + kk * 16 + (lane >> 4) * 8) * 2), a[0], a[1],
                    a[2], a[3]);
            mma16816(s, a, qb[kk][0], qb[kk][1]);
        }
        // s[0], s[1]: token g, heads 2tq, 2tq+1; s[2], s[3]: token g + 8
        if (tok0 + g >= ctx) s[0] = s[1] = -INFINITY;
        if (tok0 + g + 8 >= ctx) s[2] = s[3] = -INFINITY;
        float mt[2] = {fmaxf(s[0], s[2]), fmaxf(s[1], s[3])};
        float alpha[2];
#pragma unroll
        for (int hc = 0; hc < 2; ++hc) {
            mt[hc] = fmaxf(mt[hc], __shfl_xor_sync(0xffffffffu, mt[hc], 4));
            mt[hc] = fmaxf(mt[hc], __shfl_xor_sync(0xffffffffu, mt[hc], 8));
            mt[hc] = fmaxf(mt[hc], __shfl_xor_sync(0xffffffffu, mt[hc], 16));
            const float mn = fmaxf(m_run[hc], mt[hc]);
            alpha[hc] = mn == -INFINITY ? 1.f : exp2f(m_run[hc] - mn);
            m_run[hc] = mn;
        }
#pragma unroll
        for (int e = 0; e < 4; ++e) s[e] = m_run[e & 1] == -INFINITY ? 0.f : exp2f(s[e] - m_run[e & 1]);
        l_run[0] = l_run[0] * alpha[0] + s[0] + s[2];
        l_run[1] = l_run[1] * alpha[1] + s[1] + s[3];
        if (__any_sync(0xffffffffu, alpha[0] != 1.f || alpha[1] != 1.f)) {
#pragma unroll
            for (int mt2 = 0; mt2 < KS; ++mt2) {
                acc[mt2][0] *= alpha[0];
                acc[mt2][1] *= alpha[1];
                acc[mt2][2] *= alpha[0];
                acc[mt2][3] *= alpha[1];
            }
        }
        // P^T (k = token, n = head) as the B operand: transpose the two 8x8 token halves
        const uint32_t pb0 = movmatrix_t(pack2(s[0], s[1]));
        const uint32_t pb1 = movmatrix_t(pack2(s[2], s[3]));
        const uint32_t vbase = smem_u32(&sm.v[warp][buf][0][0]);
#pragma unroll
        for (int mt2 = 0; mt2 < KS; ++mt2) {
            uint32_t a[4];
            // A = V^T (dims x tokens) from V [token][dim] with the transposing ldmatrix
            ldsm_x4_t(vbase + uint32_t((((lane & 7) + ((lane >> 4) & 1) * 8) * (DH + 8) + mt2 * 16 +
                                        ((lane >> 3) & 1) * 8) * 2),
                      a[0], a[1], a[2], a[3]);
            mma16816(acc[mt2], a, pb0, pb1);
        }
        __syncwarp();
    }
    cp_async_wait<0>();
#pragma unroll
    for (int hc = 0; hc < 2; ++hc) {  // row sums: over the tokens held by the 8 g-lanes
        l_run[hc] += __shfl_xor_sync(0xffffffffu, l_run[hc], 4);
        l_run[hc] += __shfl_xor_sync(0xffffffffu, l_run[hc], 8);
        l_run[hc] += __shfl_xor_sync(0xffffffffu, l_run[hc], 16);
    }
    // merge the 4 warps' states through shared memory: red[warp][head 8][DH + 2]
    __syncthreads();
    float* red = reinterpret_cast<float*>(&sm.k[0][0][0][0]);
#pragma unroll
    for (int mt2 = 0; mt2 < KS; ++mt2)
#pragma unroll
        for (int e = 0; e < 4; ++e) {
            const int h = 2 * tq + (e & 1), dd = mt2 * 16 + g + ((e & 2) ? 8 : 0);
            red[(warp * 8 + h) * (DH + 2) + dd] = acc[mt2][e];
        }
    if (g == 0) {
#pragma unroll
        for (int hc = 0; hc < 2; ++hc) {
            red[(warp * 8 + 2 * tq + hc) * (DH + 2) + DH] = m_run[hc];
            red[(warp * 8 + 2 * tq + hc) * (DH + 2) + DH + 1] = l_run[hc];
        }
    }
    __syncthreads();
    for (int i = threadIdx.x; i < G * DH; i += blockDim.x) {
        const int r = i / DH, dd = i % DH;
        float M = -INFINITY;
#pragma unroll
        for (int w = 0; w < kAttnWarps; ++w) M = fmaxf(M, red[(w * 8 + r) * (DH + 2) + DH]);
        float num = 0.f, den = 0.f;
#pragma unroll
        for (int w = 0; w < kAttnWarps; ++w) {
            const float* src = red + (w * 8 + r) * (DH + 2);
            const float wt = src[DH] == -INFINITY ? 0.f : exp2f(src[DH] - M);
            num += src[dd] * wt;
            den += src[DH + 1] * wt;
        }
        const size_t row_head = size_t(t) * n_h + kvh * G + r;
        if (splits == 1) {
            o[row_head * DH + dd] = f2bf(num / den);
        } else {
            float* dst = ws + (row_head * stride + split) * (DH + 2);
            __stcg(dst + dd, num);
            if (dd == 0) {
                __stcg(dst + DH, M);
                __stcg(dst + DH + 1, den);
            }
        }
    }
    if (splits == 1) return;
    __threadfence();
    __syncthreads();
    __shared__ int last_cta;
    if (threadIdx.x == 0) {
        int* cnt = counters + size_t(t) * n_kv + kvh;
        const int old = atomicAdd(cnt, 1);
        last_cta = old == splits - 1;
        if (last_cta) *cnt = 0;
    }
    __syncthreads();
    if (!last_cta) return;
    __threadfence();
    for (int i = threadIdx.x; i < G * DH; i += blockDim.x) {
        const int r = i / DH, dd = i % DH;
        const size_t row_head = size_t(t) * n_h + kvh * G + r;
        const float* base = ws + row_head * stride * (DH + 2);
        float M = -INFINITY;
        for (int sp = 0; sp < splits; ++sp) M = fmaxf(M, __ldcg(base + sp * (DH + 2) + DH));
        float num = 0.f, den = 0.f;
        for (int sp = 0; sp < splits; ++sp) {
            const float ms = __ldcg(base + sp * (DH + 2) + DH);
            if (ms == -INFINITY) continue;
            const float w = exp2f(ms - M);
            num += __ldcg(base + sp * (DH + 2) + dd) * w;
            den += __ldcg(base + sp * (DH + 2) + DH + 1) * w;
        }
        o[row_head * DH + dd] = f2bf(num / den);
    }
}

// TMA-staged variant of attn_decode_t_kernel (the default for d_head 64 / 128, G <= 8): each
// warp's ring slots are filled by cp.async.bulk.tensor loads of its 16-token K and V chunks
// (16 rows x 64 elements per box, 128-byte swizzle: conflict-free ldmatrix without padding)
// completing on a per-slot mbarrier -- one elected lane issues 2 * DH/64 bulk copies per chunk
// instead of 32 lanes x 16 cp.async, and the copy engine streams them. Same operand-swapped
// MMAs, online softmax, warp merge and split merge as attn_decode_t_kernel.
template <int DH, int ST>
struct DecTmaSmem {
    static constexpr int kBox = kDecChunk * 64;  // elements of one 16 x 64 box (2 KB)
    static constexpr int kChunk = DH / 64 * kBox;
    alignas(1024) __nv_bfloat16 k[kAttnWarps][ST][kChunk];
    alignas(1024) __nv_bfloat16 v[kAttnWarps][ST][kChunk];
    uint64_t bar[kAttnWarps][ST];
};

// byte offset of (row, 16-byte chunk c over the d_head elements) in a chunk of 64-element boxes
DS_DEVICE uint32_t swz_off(int row, int c) {
    return uint32_t((c >> 3) * (kDecChunk * 128) + row * 128 + (((c & 7) ^ (row & 7)) << 4));
}


template <int DH, int ST>
__global__ void __launch_bounds__(kAttnWarps * 32)
attn_decode_tma_kernel(const __grid_constant__ CUtensorMap tmap_kv, const __nv_bfloat16* __restrict__ q,
                       int n_h, const int32_t* __restrict__ row_pos,
                       const int32_t* __restrict__ row_page_off, const int32_t* __restrict__ flat_pages,
                       const int32_t* __restrict__ drows, KvLayout kv, int layer, int splits, int stride,
                       __nv_bfloat16* __restrict__ o, float* __restrict__ ws, int* __restrict__ counters) {
    pdl_launch_dependents();
    extern __shared__ __align__(1024) uint8_t dec_smem_raw[];
    DecTmaSmem<DH, ST>& sm = *reinterpret_cast<DecTmaSmem<DH, ST>*>(
        (reinterpret_cast<uintptr_t>(dec_smem_raw) + 1023) & ~uintptr_t(1023));
    constexpr int KS = DH / 16;
    constexpr uint32_t kChunkBytes = uint32_t(2 * kDecChunk * DH * 2);  // K + V
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    if (lane == 0) {
        tma_prefetch_desc(&tmap_kv);
#pragma unroll
        for (int b = 0; b < ST; ++b) mbar_init(&sm.bar[warp][b], 1);
        fence_mbar_init();
    }
    __syncwarp();
    pdl_wait();
    const int n_kv = kv.n_kv;
    const int G = n_h / n_kv;
    const int split = blockIdx.x % splits;
    const int kvh = (blockIdx.x / splits) % n_kv;
    const int t = drows[blockIdx.x / (splits * n_kv)];
    const int g = lane >> 2, tq = lane & 3;
    const int ctx = row_pos[t] + 1;
    const int n_chunks = (ctx + kDecChunk - 1) / kDecChunk;
    const int ch0 = split * n_chunks / splits, ch1 = (split + 1) * n_chunks / splits;
    const int32_t* pages = flat_pages + row_page_off[t];

    uint32_t qb[KS][2];
    const float qs = rsqrtf(float(DH)) * 1.4426950408889634f;
#pragma unroll
    for (int kk = 0; kk < KS; ++kk)
#pragma unroll
        for (int i = 0; i < 2; ++i) {
            float x0 = 0.f, x1 = 0.f;
            if (g < G) {
                const __nv_bfloat162 v2 = *reinterpret_cast<const __nv_bfloat162*>(
                    q + (size_t(t) * n_h + kvh * G + g) * DH + kk * 16 + 2 * tq + 8 * i);
                x0 = __bfloat162float(v2.x) * qs;
                x1 = __bfloat162float(v2.y) * qs;
            }
            qb[kk][i] = pack2(x0, x1);
        }
    float m_run[2] = {-INFINITY, -INFINITY}, l_run[2] = {0.f, 0.f};
    float acc[KS][4];
#pragma unroll
    for (int j = 0; j < KS; ++j) acc[j][0] = acc[j][1] = acc[j][2] = acc[j][3] = 0.f;

    // TMA rows of token 0 of this (layer, kv head) K / V block within a page
    const int row_k = (layer * 2 + 0) * n_kv + kvh;
    const int row_v = (layer * 2 + 1) * n_kv + kvh;
    const int rows_per_page = kv.n_layers * 2 * n_kv * 256;
    const int my_n = ch1 - ch0 > warp ? (ch1 - ch0 - warp + kAttnWarps - 1) / kAttnWarps : 0;
    auto load = [&](int j, int buf) {  // lane 0 only
        const int tok0 = (ch0 + warp + j * kAttnWarps) * kDecChunk;
        const int base = pages[tok0 >> 8] * rows_per_page + (tok0 & 255);
        uint64_t* bar = &sm.bar[warp][buf];
        fence_proxy_async_smem();  // generic reads / zero-fill of this slot precede the refill
        mbar_arrive_expect_tx(bar, kChunkBytes);
#pragma unroll
        for (int bx = 0; bx < DH / 64; ++bx) {
            tma_load_2d(&sm.k[warp][buf][bx * DecTmaSmem<DH, ST>::kBox], &tmap_kv, bar, bx * 64, base + row_k * 256);
            tma_load_2d(&sm.v[warp][buf][bx * DecTmaSmem<DH, ST>::kBox], &tmap_kv, bar, bx * 64, base + row_v * 256);
        }
    };
    if (lane == 0) {
#pragma unroll
        for (int j = 0; j < ST - 1; ++j)
            if (j < my_n) load(j, j);
    }
    for (int j = 0; j < my_n; ++j) {
        const int buf = j % ST;
        if (lane == 0 && j + ST - 1 < my_n) load(j + ST - 1, (j + ST - 1) % ST);
        mbar_wait(&sm.bar[warp][buf], uint32_t((j / ST) & 1));
        const int tok0 = (ch0 + warp + j * kAttnWarps) * kDecChunk;
        const int valid = min(kDecChunk, ctx - tok0);
        const uint32_t kbase = smem_u32(&sm.k[warp][buf][0]);
        const uint32_t vbase = smem_u32(&sm.v[warp][buf][0]);
        if (valid < kDecChunk) {  // rows past the context: zero V (no 0 * garbage = NaN)
            uint8_t* vb = reinterpret_cast<uint8_t*>(&sm.v[warp][buf][0]);
            for (int i = lane; i < (kDecChunk - valid) * (DH / 8); i += 32) {
                const int r = valid + i / (DH / 8), c = i % (DH / 8);
                *reinterpret_cast<uint4*>(vb + swz_off(r, c)) = make_uint4(0, 0, 0, 0);
            }
            __syncwarp();
        }
        float s[4] = {0.f, 0.f, 0.f, 0.f};
#pragma unroll
        for (int kk = 0; kk < KS; ++kk) {
            uint32_t a[4];
            ldsm_x4(kbase + swz_off(lane & 15, kk * 2 + (lane >> 4)), a[0], a[1], a[2], a[3]);
            mma16816(s, a, qb[kk][0], qb[kk][1]);
        }
        if (tok0 + g >= ctx) s[0] = s[1] = -INFINITY;
        if (tok0 + g + 8 >= ctx) s[2] = s[3] = -INFINITY;
        float mt[2] = {fmaxf(s[0], s[2]), fmaxf(s[1], s[3])};
        float alpha[2];
#pragma unroll
        for (int hc = 0; hc < 2; ++hc) {
            mt[hc] = fmaxf(mt[hc], __shfl_xor_sync(0xffffffffu, mt[hc], 4));
            mt[hc] = fmaxf(mt[hc], __shfl_xor_sync(0xffffffffu, mt[hc], 8));
            mt[hc] = fmaxf(mt[hc], __shfl_xor_sync(0xffffffffu, mt[hc], 16));
            const float mn = fmaxf(m_run[hc], mt[hc]);
            alpha[hc] = mn == -INFINITY ? 1.f : exp2f(m_run[hc] - mn);
            m_run[hc] = mn;
        }
#pragma unroll
        for (int e = 0; e < 4; ++e) s[e] = m_run[e & 1] == -INFINITY ? 0.f : exp2f(s[e] - m_run[e & 1]);
        l_run[0] = l_run[0] * alpha[0] + s[0] + s[2];
        l_run[1] = l_run[1] * alpha[1] + s[1] + s[3];
        if (__any_sync(0xffffffffu, alpha[0] != 1.f || alpha[1] != 1.f)) {
#pragma unroll
            for (int mt2 = 0; mt2 < KS; ++mt2) {
                acc[mt2][0] *= alpha[0];
                acc[mt2][1] *= alpha[1];
                acc[mt2][2] *= alpha[0];
                acc[mt2][3] *= alpha[1];
            }
        }
        const uint32_t pb0 = movmatrix_t(pack2(s[0], s[1]));
        const uint32_t pb1 = movmatrix_t(pack2(s[2], s[3]));
#pragma unroll
        for (int mt2 = 0; mt2 < KS; ++mt2) {
            uint32_t a[4];
            ldsm_x4_t(vbase + swz_off((lane & 7) + ((lane >> 4) & 1) * 8, mt2 * 2 + ((lane >> 3) & 1)),
                      a[0], a[1], a[2], a[3]);
            mma16816(acc[mt2], a, pb0, pb1);
        }
        __syncwarp();
    }
#pragma unroll
    for (int hc = 0; hc < 2; ++hc) {
        l_run[hc] += __shfl_xor_sync(0xffffffffu, l_run[hc], 4);
        l_run[hc] += __shfl_xor_sync(0xffffffffu, l_run[hc], 8);
        l_run[hc] += __shfl_xor_sync(0xffffffffu, l_run[hc], 16);
    }
    __syncthreads();  // every warp's bulk copies have landed (waited) before the slots are reused
    float* red = reinterpret_cast<float*>(&sm.k[0][0][0]);
#pragma unroll
    for (int mt2 = 0; mt2 < KS; ++mt2)
#pragma unroll
        for (int e = 0; e < 4; ++e) {
            const int h = 2 * tq + (e & 1), dd = mt2 * 16 + g + ((e & 2) ? 8 : 0);
            red[(warp * 8 + h) * (DH + 2) + dd] = acc[mt2][e];
        }
    if (g == 0) {
#pragma unroll
        for (int hc = 0; hc < 2; ++hc) {
            red[(warp * 8 + 2 * tq + hc) * (DH + 2) + DH] = m_run[hc];
            red[(warp * 8 + 2 * tq + hc) * (DH + 2) + DH + 1] = l_run[hc];
        }
    }
    __syncthreads();
    for (int i = threadIdx.x; i < G * DH; i += blockDim.x) {
        const int r = i / DH, dd = i % DH;
        float M = -INFINITY;
#pragma unroll
        for (int w = 0; w < kAttnWarps; ++w) M = fmaxf(M, red[(w * 8 + r) * (DH + 2) + DH]);
        float num = 0.f, den = 0.f;
#pragma unroll
        for (int w = 0; w < kAttnWarps; ++w) {
            const float* src = red + (w * 8 + r) * (DH + 2);
            const float wt = src[DH] == -INFINITY ? 0.f : exp2f(src[DH] - M);
            num += src[dd] * wt;
            den += src[DH + 1] * wt;
        }
        const size_t row_head = size_t(t) * n_h + kvh * G + r;
        if (splits == 1) {
            o[row_head * DH + dd] = f2bf(num / den);
        } else {
            float* dst = ws + (row_head * stride + split) * (DH + 2);
            __stcg(dst + dd, num);
            if (dd == 0) {
                __stcg(dst + DH, M);
                __stcg(dst + DH + 1, den);
            }
        }
    }
    if (splits == 1) return;
    __threadfence();
    __syncthreads();
    __shared__ int last_cta;
    if (threadIdx.x == 0) {
        int* cnt = counters + size_t(t) * n_kv + kvh;
        const int old = atomicAdd(cnt, 1);
        last_cta = old == splits - 1;
        if (last_cta) *cnt = 0;
    }
    __syncthreads();
    if (!last_cta) return;
    __threadfence();
    for (int i = threadIdx.x; i < G * DH; i += blockDim.x) {
        const int r = i / DH, dd = i % DH;
        const size_t row_head = size_t(t) * n_h + kvh * G + r;
        const float* base = ws + row_head * stride * (DH + 2);
        float M = -INFINITY;
        for (int sp = 0; sp < splits; ++sp) M = fmaxf(M, __ldcg(base + sp * (DH + 2) + DH));
        float num = 0.f, den = 0.f;
        for (int sp = 0; sp < splits; ++sp) {
            const float ms = __ldcg(base + sp * (DH + 2) + DH);
            if (ms == -INFINITY) continue;
            const float w = exp2f(ms - M);
            num += __ldcg(base + sp * (DH + 2) + dd) * w;
            den += __ldcg(base + sp * (DH + 2) + DH + 1) * w;
        }
        o[row_head * DH + dd] = f2bf(num / den);
    }
}

// timing experiments only (results invalid): DS_TC_DBG bit 0 no exp2, 1 no PV MMAs, 2 no S MMAs,
// 3 no K/V loads
static int tc_dbg() {
    static const int v = getenv("DS_TC_DBG") ? atoi(getenv("DS_TC_DBG")) : 0;
    return v;
}
// DS_ATTN_PROMPT: 1 cp.async-staged mma.sync kernel, 2 TMA-staged mma.sync kernel, 3 (default)
// tcgen05 kernel where it applies (d_head 128, G <= 8, no prompt context splits; 128-row query
// blocks), else 2
static int prompt_kernel_env() {
    static const int v = getenv("DS_ATTN_PROMPT") ? atoi(getenv("DS_ATTN_PROMPT")) : 3;
    return v;
}
static bool prompt_tc(int n_h, int n_kv, int d_head) {
    static const int sp_tiles = getenv("DS_ATTN_PROMPT_TILES") ? atoi(getenv("DS_ATTN_PROMPT_TILES")) : 0;
    const int G = n_h / n_kv;
    return prompt_kernel_env() == 3 && d_head == 128 && (G == 1 || G == 2 || G == 4 || G == 8) && sp_tiles == 0;
}
int attention_block_positions(int n_h, int n_kv, int d_head) {
    if (prompt_tc(n_h, n_kv, d_head)) return kTcRows / (n_h / n_kv);
    return (kAttnWarps * 16) / (n_h / n_kv);
}

// Context splits (flash-decoding): at least kSplitTarget CTAs per SM when the (block, kv head)
// count alone is short of that, each split keeping >= 2 tiles (128 tokens) of the longest context.
static int split_target() {
    // 1 CTA per SM of (row, KV head) work before splitting (measured on config 2: targets 0 / 1 /
    // 2 / 3 -> 4786 / 4796 / 4953 / 4988 ms per step with the operand-swapped decode kernel)
    static const int v = getenv("DS_ATTN_TARGET") ? atoi(getenv("DS_ATTN_TARGET")) : 1;
    return v;
}
int attention_pick_splits(int n_blocks, int n_kv, int max_ctx) {
    const int base = n_blocks * n_kv;
    const int tiles = (max_ctx + kTile - 1) / kTile;
    int s = (split_target() * kNumSMs + base - 1) / base;
    if (s > tiles / 2) s = tiles / 2;
    if (s > 16) s = 16;
    return s < 1 ? 1 : s;
}

// Context splits: decode rows by the CTA-count heuristic above; prompt blocks so that no CTA
// walks more than 2 tiles (128 tokens) of the longest context (their mma.sync work, not HBM,
// bounds a long prompt chunk). Both shrink until T x max(splits) partials fit the workspace.
void attention_splits(int T, int n_h, int d_head, int n_blocks, int n_drows, int n_kv, int max_ctx,
                      int max_prompt_ctx, size_t ws_floats, int* s_prompt, int* s_decode) {
    int sd = n_drows > 0 ? attention_pick_splits(n_blocks + n_drows, n_kv, max_ctx) : 1;
    const int tiles = (max_prompt_ctx + kTile - 1) / kTile;
    // prompt blocks: unsplit by default. DS_ATTN_PROMPT_TILES=n caps a CTA at n tiles; measured
    // 0.5-0.8 s slower per config-2 step at n = 2..4: the last CTA's merge of 64 rows x d_head
    // over the splits costs more than the shorter tile chain saves
    static const int sp_tiles = getenv("DS_ATTN_PROMPT_TILES") ? atoi(getenv("DS_ATTN_PROMPT_TILES")) : 0;
    int sp = (n_blocks > 0 && sp_tiles > 0) ? std::min(8, std::max(1, (tiles + sp_tiles - 1) / sp_tiles)) : 1;
    while (std::max(sp, sd) > 1 && attention_workspace_floats(T, n_h, d_head, std::max(sp, sd)) > ws_floats) {
        if (sp >= sd) --sp; else --sd;
    }
    *s_prompt = sp;
    *s_decode = sd;
}

int attention_launches(int n_blocks, int n_drows, int s_prompt, int s_decode) {
    if (n_blocks + n_drows <= 0) return 0;
    (void)s_prompt;
    (void)s_decode;
    return (n_blocks > 0) + (n_drows > 0);
}

size_t attention_workspace_floats(int T, int n_h, int d_head, int splits) {
    return size_t(T) * n_h * splits * (d_head + 2);
}

// Decode ring depth (DS_ATTN_STAGES=2|3|4 for tuning experiments; default kDecStages).
static int decode_stages() {
    static const int st = [] {
        const char* e = getenv("DS_ATTN_STAGES");
        const int v = e ? atoi(e) : kDecStages;
        return (v >= 2 && v <= 4) ? v : kDecStages;
    }();
    return st;
}

template <int DH>
static void launch(const __nv_bfloat16* q, int T, int n_h, const int32_t* row_pos,
                   const int32_t* row_page_off, const int32_t* flat_pages, const int32_t* blocks,
                   int n_blocks, const int32_t* drows, int n_drows,
                   const KvLayout& kv, int layer, int sp, int sd, __nv_bfloat16* o, float* ws,
                   int* counters, const L2Prefetch& pf, cudaStream_t stream) {
    const L2Prefetch pf_dec = pf;  // the decode launch (or the prompt one when alone) prefetches
    // timing experiments only (results invalid): DS_ATTN_SKIP bit 0 prompt blocks, 1 decode rows
    static const int skip = getenv("DS_ATTN_SKIP") ? atoi(getenv("DS_ATTN_SKIP")) : 0;
    if (skip & 1) n_blocks = 0;
    if (skip & 2) n_drows = 0;
    const int stride = std::max(sp, sd);
    const int prompt_env = prompt_kernel_env();
    if (n_blocks > 0 && prompt_tc(n_h, kv.n_kv, DH) && kv.tmap64) {
        const CUtensorMap& tk = *static_cast<const CUtensorMap*>(kv.tmap64);
        const dim3 g(n_blocks * kv.n_kv), b(384);
        const size_t sm_bytes = sizeof(PromptTcSmem) + 1024;
        switch (n_h / kv.n_kv) {
            case 1: launch_pdl(attn_prompt_tc_kernel<1>, g, b, sm_bytes, stream, tk, q, n_h, row_pos, row_page_off, flat_pages, blocks, kv, layer, o, tc_dbg()); break;
            case 2: launch_pdl(attn_prompt_tc_kernel<2>, g, b, sm_bytes, stream, tk, q, n_h, row_pos, row_page_off, flat_pages, blocks, kv, layer, o, tc_dbg()); break;
            case 4: launch_pdl(attn_prompt_tc_kernel<4>, g, b, sm_bytes, stream, tk, q, n_h, row_pos, row_page_off, flat_pages, blocks, kv, layer, o, tc_dbg()); break;
            default: launch_pdl(attn_prompt_tc_kernel<8>, g, b, sm_bytes, stream, tk, q, n_h, row_pos, row_page_off, flat_pages, blocks, kv, layer, o, tc_dbg()); break;
        }
    } else if (n_blocks > 0 && prompt_env >= 2 && kv.tmap64)
        launch_pdl(attn_prompt_tma_kernel<DH>, dim3(n_blocks * kv.n_kv * sp), dim3(kPromptWarps * 32),
                   sizeof(PromptTmaSmem<DH>) + 1024, stream, *static_cast<const CUtensorMap*>(kv.tmap64), q,
                   n_h, row_pos, row_page_off, flat_pages, blocks, kv, layer, sp, stride, o, ws,
                   counters + size_t(T) * kv.n_kv);
    else if (n_blocks > 0)
        launch_pdl(attn_prompt_kernel<DH>, dim3(n_blocks * kv.n_kv * sp), dim3(kPromptWarps * 32),
                   sizeof(PromptSmem<DH>), stream, q, n_h, row_pos, row_page_off, flat_pages, blocks,
                   kv, layer, sp, stride, o, ws, counters + size_t(T) * kv.n_kv,
                   n_drows > 0 ? L2Prefetch{} : pf);
    if (n_drows > 0) {
        const dim3 grid(n_drows * kv.n_kv * sd), block(kAttnWarps * 32);
        // ring depth by occupancy: a grid of <= 1 (2) CTA per SM keeps the same 12 chunks in
        // flight per SM with 4- (3-) deep rings that 3 resident CTAs get with 2-deep ones
        int st = decode_stages();
        if (st == kDecStages && getenv("DS_ATTN_STAGES") == nullptr) {
            const int ctas = int(grid.x);
            st = ctas <= kNumSMs ? 4 : (ctas <= 2 * kNumSMs ? 3 : 2);
        }
        // TMA-staged operand-swapped kernel for G <= 8 (DS_ATTN_DECODE=3, the default when the
        // pool has a tensor map); 2: the same MMAs staged with cp.async; 1: the Q-as-M kernel
        static const int dec_env = getenv("DS_ATTN_DECODE") ? atoi(getenv("DS_ATTN_DECODE")) : 3;
        if (dec_env == 3 && n_h / kv.n_kv <= 8 && kv.tmap) {
            const CUtensorMap& tm = *static_cast<const CUtensorMap*>(kv.tmap);
            switch (st) {
                case 3:
                    launch_pdl(attn_decode_tma_kernel<DH, 3>, grid, block, sizeof(DecTmaSmem<DH, 3>) + 1024,
                               stream, tm, q, n_h, row_pos, row_page_off, flat_pages, drows, kv, layer, sd,
                               stride, o, ws, counters);
                    break;
                case 4:
                    launch_pdl(attn_decode_tma_kernel<DH, 4>, grid, block, sizeof(DecTmaSmem<DH, 4>) + 1024,
                               stream, tm, q, n_h, row_pos, row_page_off, flat_pages, drows, kv, layer, sd,
                               stride, o, ws, counters);
                    break;
                default:
                    launch_pdl(attn_decode_tma_kernel<DH, 2>, grid, block, sizeof(DecTmaSmem<DH, 2>) + 1024,
                               stream, tm, q, n_h, row_pos, row_page_off, flat_pages, drows, kv, layer, sd,
                               stride, o, ws, counters);
            }
            return;
        }
        if (dec_env == 2 && n_h / kv.n_kv <= 8) {
            switch (st) {
                case 3:
                    launch_pdl(attn_decode_t_kernel<DH, 3>, grid, block, sizeof(DecSmem<DH, 3>), stream, q,
                               n_h, row_pos, row_page_off, flat_pages, drows, kv, layer, sd, stride, o, ws,
                               counters, pf_dec);
                    break;
                case 4:
                    launch_pdl(attn_decode_t_kernel<DH, 4>, grid, block, sizeof(DecSmem<DH, 4>), stream, q,
                               n_h, row_pos, row_page_off, flat_pages, drows, kv, layer, sd, stride, o, ws,
                               counters, pf_dec);
                    break;
                default:
                    launch_pdl(attn_decode_t_kernel<DH, 2>, grid, block, sizeof(DecSmem<DH, 2>), stream, q,
                               n_h, row_pos, row_page_off, flat_pages, drows, kv, layer, sd, stride, o, ws,
                               counters, pf_dec);
            }
            return;
        }
        switch (st) {
            case 3:
                launch_pdl(attn_decode_kernel<DH, 3>, grid, block, sizeof(DecSmem<DH, 3>), stream, q,
                           n_h, row_pos, row_page_off, flat_pages, drows, kv, layer, sd, stride, o, ws,
                           counters, pf_dec);
                break;
            case 4:
                launch_pdl(attn_decode_kernel<DH, 4>, grid, block, sizeof(DecSmem<DH, 4>), stream, q,
                           n_h, row_pos, row_page_off, flat_pages, drows, kv, layer, sd, stride, o, ws,
                           counters, pf_dec);
                break;
            default:
                launch_pdl(attn_decode_kernel<DH, 2>, grid, block, sizeof(DecSmem<DH, 2>), stream, q,
                           n_h, row_pos, row_page_off, flat_pages, drows, kv, layer, sd, stride, o, ws,
                           counters, pf_dec);
        }
    }
}

int attention_paged(const __nv_bfloat16* q, int T, int n_h, const int32_t* row_pos,
                    const int32_t* row_page_off, const int32_t* flat_pages, const int32_t* blocks,
                    int n_blocks, const int32_t* drows, int n_drows,
                    const KvLayout& kv, int layer, int s_prompt, int s_decode, __nv_bfloat16* o,
                    float* ws, size_t ws_floats, int* counters, const L2Prefetch& pf,
                    cudaStream_t stream) {
    if (T <= 0 || n_blocks + n_drows <= 0) return 0;
    if (n_h % kv.n_kv != 0 || n_h / kv.n_kv > 16) return -1;
    if (attention_workspace_floats(T, n_h, kv.d_head, std::max(s_prompt, s_decode)) > ws_floats &&
        std::max(s_prompt, s_decode) > 1)
        return -4;
    if (kv.d_head == 128)
        launch<128>(q, T, n_h, row_pos, row_page_off, flat_pages, blocks, n_blocks, drows, n_drows,
                    kv, layer, s_prompt, s_decode, o, ws, counters, pf, stream);
    else if (kv.d_head == 64)
        launch<64>(q, T, n_h, row_pos, row_page_off, flat_pages, blocks, n_blocks, drows, n_drows,
                   kv, layer, s_prompt, s_decode, o, ws, counters, pf, stream);
    else
        return -2;
    return cudaPeekAtLastError() == cudaSuccess ? 0 : -3;
}
}  // namespace ds

namespace ds {
template <int DH, int ST>
static void preload_decode() {
    cudaFuncAttributes a;
    cudaFuncGetAttributes(&a, attn_decode_tma_kernel<DH, ST>);
    cudaFuncSetAttribute(attn_decode_tma_kernel<DH, ST>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                         int(sizeof(DecTmaSmem<DH, ST>) + 1024));
    cudaFuncGetAttributes(&a, attn_decode_kernel<DH, ST>);
    cudaFuncSetAttribute(attn_decode_kernel<DH, ST>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                         int(sizeof(DecSmem<DH, ST>)));
    cudaFuncGetAttributes(&a, attn_decode_t_kernel<DH, ST>);
    cudaFuncSetAttribute(attn_decode_t_kernel<DH, ST>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                         int(sizeof(DecSmem<DH, ST>)));
}

template <int G>
static void preload_prompt_tc() {
    cudaFuncAttributes a;
    cudaFuncGetAttributes(&a, attn_prompt_tc_kernel<G>);
    cudaFuncSetAttribute(attn_prompt_tc_kernel<G>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                         int(sizeof(PromptTcSmem) + 1024));
}

void preload_attention() {
    preload_prompt_tc<1>();
    preload_prompt_tc<2>();
    preload_prompt_tc<4>();
    preload_prompt_tc<8>();
    cudaFuncAttributes a;
    cudaFuncGetAttributes(&a, attn_prompt_tma_kernel<128>);
    cudaFuncGetAttributes(&a, attn_prompt_tma_kernel<64>);
    cudaFuncSetAttribute(attn_prompt_tma_kernel<128>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                         int(sizeof(PromptTmaSmem<128>) + 1024));
    cudaFuncSetAttribute(attn_prompt_tma_kernel<64>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                         int(sizeof(PromptTmaSmem<64>) + 1024));
    cudaFuncGetAttributes(&a, attn_prompt_kernel<128>);
    cudaFuncGetAttributes(&a, attn_prompt_kernel<64>);
    cudaFuncSetAttribute(attn_prompt_kernel<128>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                         int(sizeof(PromptSmem<128>)));
    cudaFuncSetAttribute(attn_prompt_kernel<64>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                         int(sizeof(PromptSmem<64>)));
    preload_decode<128, 2>();
    preload_decode<128, 3>();
    preload_decode<128, 4>();
    preload_decode<64, 2>();
    preload_decode<64, 3>();
    preload_decode<64, 4>();
}
}  // namespace ds
