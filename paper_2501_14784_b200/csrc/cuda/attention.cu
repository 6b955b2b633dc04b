// Paged causal GQA attention over the stage's KV pages (decode rows and chunked-prefill rows in
// one launch). CTA = (row, kv-head, context split); the K/V tiles of 64 tokens (never straddling
// a 256-token page) are staged in shared memory with 16-byte coalesced loads, the G = n_h/n_kv
// query heads of the group share every staged tile (GQA reuse), and each warp keeps an online
// softmax (log2 domain, fp32) per head. Context splits (flash-decoding) keep >= 2 CTAs per SM
// when the row count is small; a combine kernel merges the (o, m, l) partials.
//
// HBM roofline: each CTA reads ctx * d_head * 2 (K,V) * 2 B once; bytes/row/layer = ctx * 4 *
// n_kv * d_head.
#include "common.cuh"
#include "kernels.h"

namespace ds {

constexpr int kAttnTile = 64;
constexpr int kAttnThreads = 128;

template <int DH>
struct AttnSmem {
    __nv_bfloat16 k[kAttnTile][DH + 8];
    __nv_bfloat16 v[kAttnTile][DH + 8];
    float q[8][DH];
};

template <int DH>
__global__ void __launch_bounds__(kAttnThreads)
attn_kernel(const __nv_bfloat16* __restrict__ q, int n_h, const int32_t* __restrict__ row_pos,
            const int32_t* __restrict__ row_page_off, const int32_t* __restrict__ flat_pages,
            KvLayout kv, int layer, int splits, __nv_bfloat16* __restrict__ o, float* __restrict__ ws) {
    __shared__ __align__(16) AttnSmem<DH> sm;
    const int n_kv = kv.n_kv;
    const int G = n_h / n_kv;
    const int split = blockIdx.x % splits;
    const int kvh = (blockIdx.x / splits) % n_kv;
    const int t = blockIdx.x / (splits * n_kv);
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;

    const int ctx = row_pos[t] + 1;
    const int n_tiles = (ctx + kAttnTile - 1) / kAttnTile;
    const int tile0 = split * n_tiles / splits;
    const int tile1 = (split + 1) * n_tiles / splits;
    const int32_t* pages = flat_pages + row_page_off[t];

    // q heads of this group, pre-scaled into the log2 domain
    const float qscale = rsqrtf(float(DH)) * 1.4426950408889634f;
    for (int i = threadIdx.x; i < G * DH; i += blockDim.x) {
        const int h = i / DH, dd = i % DH;
        sm.q[h][dd] = bf2f(q[(size_t(t) * n_h + kvh * G + h) * DH + dd]) * qscale;
    }

    constexpr int DPL = DH / 32;  // output dims per lane
    float m[2], l[2], acc[2][DPL];
#pragma unroll
    for (int i = 0; i < 2; ++i) {
        m[i] = -INFINITY;
        l[i] = 0.f;
#pragma unroll
        for (int j = 0; j < DPL; ++j) acc[i][j] = 0.f;
    }

    const size_t kv_head_off_k = ((size_t(layer) * 2 + 0) * n_kv + kvh) * 256 * DH;
    const size_t kv_head_off_v = ((size_t(layer) * 2 + 1) * n_kv + kvh) * 256 * DH;
    constexpr int VEC_PER_ROW = DH / 8;

    for (int tile = tile0; tile < tile1; ++tile) {
        const int tok0 = tile * kAttnTile;
        const size_t page_base = size_t(pages[tok0 >> 8]) * kv.page_elems + size_t(tok0 & 255) * DH;
        const uint4* ksrc = reinterpret_cast<const uint4*>(kv.pool + page_base + kv_head_off_k);
        const uint4* vsrc = reinterpret_cast<const uint4*>(kv.pool + page_base + kv_head_off_v);
        __syncthreads();  // previous tile fully consumed (and q staged on the first pass)
        for (int i = threadIdx.x; i < kAttnTile * VEC_PER_ROW; i += blockDim.x) {
            const int r = i / VEC_PER_ROW, c = i % VEC_PER_ROW;
            *reinterpret_cast<uint4*>(&sm.k[r][c * 8]) = ksrc[i];
            *reinterpret_cast<uint4*>(&sm.v[r][c * 8]) = vsrc[i];
        }
        __syncthreads();
        const int valid = min(kAttnTile, ctx - tok0);
#pragma unroll
        for (int hi = 0; hi < 2; ++hi) {
            const int h = warp + 4 * hi;
            if (h >= G) break;
            float s[2];
#pragma unroll
            for (int half = 0; half < 2; ++half) {
                const int j = lane + 32 * half;
                float dot = 0.f;
#pragma unroll
                for (int c = 0; c < VEC_PER_ROW; ++c) {
                    float kf[8];
                    unpack8(*reinterpret_cast<const uint4*>(&sm.k[j][c * 8]), kf);
                    const float4 q0 = *reinterpret_cast<const float4*>(&sm.q[h][c * 8]);
                    const float4 q1 = *reinterpret_cast<const float4*>(&sm.q[h][c * 8 + 4]);
                    dot += kf[0] * q0.x + kf[1] * q0.y + kf[2] * q0.z + kf[3] * q0.w + kf[4] * q1.x +
                           kf[5] * q1.y + kf[6] * q1.z + kf[7] * q1.w;
                }
                s[half] = j < valid ? dot : -INFINITY;
            }
            const float mt = warp_max(fmaxf(s[0], s[1]));
            const float mn = fmaxf(m[hi], mt);
            const float alpha = exp2f(m[hi] - mn);
            const float p0 = exp2f(s[0] - mn), p1 = exp2f(s[1] - mn);
            l[hi] = l[hi] * alpha + warp_sum(p0 + p1);
            m[hi] = mn;
#pragma unroll
            for (int j = 0; j < DPL; ++j) acc[hi][j] *= alpha;
            for (int j = 0; j < valid; ++j) {
                const float pj = __shfl_sync(0xffffffffu, j < 32 ? p0 : p1, j & 31);
                if (DPL == 4) {
                    const uint2 vv = *reinterpret_cast<const uint2*>(&sm.v[j][lane * 4]);
                    const __nv_bfloat162* vh = reinterpret_cast<const __nv_bfloat162*>(&vv);
                    const float2 a = __bfloat1622float2(vh[0]), b = __bfloat1622float2(vh[1]);
                    acc[hi][0] += pj * a.x;
                    acc[hi][1] += pj * a.y;
                    acc[hi][2] += pj * b.x;
                    acc[hi][3] += pj * b.y;
                } else {
#pragma unroll
                    for (int e = 0; e < DPL; ++e) acc[hi][e] += pj * bf2f(sm.v[j][lane * DPL + e]);
                }
            }
        }
    }

#pragma unroll
    for (int hi = 0; hi < 2; ++hi) {
        const int h = warp + 4 * hi;
        if (h >= G) break;
        const int head = kvh * G + h;
        if (splits == 1) {
            const float inv = 1.0f / l[hi];
            __nv_bfloat16* dst = o + (size_t(t) * n_h + head) * DH + lane * DPL;
#pragma unroll
            for (int e = 0; e < DPL; ++e) dst[e] = f2bf(acc[hi][e] * inv);
        } else {
            float* dst = ws + ((size_t(t) * n_h + head) * splits + split) * (DH + 2);
#pragma unroll
            for (int e = 0; e < DPL; ++e) dst[lane * DPL + e] = acc[hi][e];
            if (lane == 0) {
                dst[DH] = m[hi];
                dst[DH + 1] = l[hi];
            }
        }
    }
}

template <int DH>
__global__ void attn_combine_kernel(const float* __restrict__ ws, int n_rows_heads, int splits,
                                    __nv_bfloat16* __restrict__ o) {
    const int rh = blockIdx.x;
    const float* base = ws + size_t(rh) * splits * (DH + 2);
    float M = -INFINITY;
    for (int s = 0; s < splits; ++s) M = fmaxf(M, base[s * (DH + 2) + DH]);
    for (int dd = threadIdx.x; dd < DH; dd += blockDim.x) {
        float num = 0.f, den = 0.f;
        for (int s = 0; s < splits; ++s) {
            const float ms = base[s * (DH + 2) + DH];
            if (ms == -INFINITY) continue;
            const float w = exp2f(ms - M);
            num += base[s * (DH + 2) + dd] * w;
            den += base[s * (DH + 2) + DH + 1] * w;
        }
        o[size_t(rh) * DH + dd] = f2bf(num / den);
    }
}

static int pick_attn_splits(int T, int n_kv, int max_ctx) {
    const int base = T * n_kv;
    const int tiles = (max_ctx + kAttnTile - 1) / kAttnTile;
    int s = (2 * kNumSMs + base - 1) / base;
    if (s > tiles) s = tiles;
    if (s > 32) s = 32;
    return s < 1 ? 1 : s;
}

int attention_launches(int T, int n_kv, int max_ctx) {
    return T > 0 ? (pick_attn_splits(T, n_kv, max_ctx) > 1 ? 2 : 1) : 0;
}

size_t attention_workspace_floats(int T, int n_h, int d_head, int splits) {
    return size_t(T) * n_h * splits * (d_head + 2);
}

int attention_paged(const __nv_bfloat16* q, int T, int n_h, const int32_t* row_pos,
                    const int32_t* row_page_off, const int32_t* flat_pages, const KvLayout& kv,
                    int layer, int max_ctx, __nv_bfloat16* o, float* ws, size_t ws_floats,
                    cudaStream_t stream) {
    if (T <= 0) return 0;
    if (n_h % kv.n_kv != 0 || n_h / kv.n_kv > 8) return -1;
    int splits = pick_attn_splits(T, kv.n_kv, max_ctx);
    if (splits > 1 && attention_workspace_floats(T, n_h, kv.d_head, splits) > ws_floats) splits = 1;
    const int grid = T * kv.n_kv * splits;
    if (kv.d_head == 128) {
        attn_kernel<128><<<grid, kAttnThreads, 0, stream>>>(q, n_h, row_pos, row_page_off,
                                                            flat_pages, kv, layer, splits, o, ws);
        if (splits > 1) attn_combine_kernel<128><<<T * n_h, 128, 0, stream>>>(ws, T * n_h, splits, o);
    } else if (kv.d_head == 64) {
        attn_kernel<64><<<grid, kAttnThreads, 0, stream>>>(q, n_h, row_pos, row_page_off,
                                                           flat_pages, kv, layer, splits, o, ws);
        if (splits > 1) attn_combine_kernel<64><<<T * n_h, 64, 0, stream>>>(ws, T * n_h, splits, o);
    } else {
        return -2;
    }
    return cudaPeekAtLastError() == cudaSuccess ? 0 : -3;
}

}  // namespace ds
