// HBM-bound stage-forward kernels: weight init, embedding gather, RMSNorm (+ deferred residual),
// RoPE + paged KV append (+ deferred q/k/v epilogue), greedy argmax and the token plumbing between circuits. All vectorised
// 16-byte accesses; grids sized in multiples of the SM count where the row count allows.
// Numerics follow oracle/llama_ref.c exactly (bf16 storage, fp32 math, same rounding points).
#include <algorithm>

#include "common.cuh"
#include "kernels.h"

namespace ds {

// ------------------------------------------------------------ weights ----
DS_DEVICE uint64_t mix64(uint64_t z) {
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ULL;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBULL;
    return z ^ (z >> 31);
}

__global__ void init_weights_kernel(__nv_bfloat16* dst, uint64_t seed, uint64_t tensor_id,
                                    int64_t rows, int64_t cols, float scale, int part) {
    const int64_t n = rows * cols;
    const uint64_t base = seed + tensor_id * 0x9E3779B97F4A7C15ULL;
    for (int64_t i = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; i < n;
         i += int64_t(gridDim.x) * blockDim.x) {
        const uint64_t h = mix64(base + uint64_t(i) * 0xD1B54A32D192ED03ULL);
        const float u = float(h >> 40) * (1.0f / 16777216.0f);
        const float v = __fmul_rn(__fsub_rn(__fmul_rn(2.0f, u), 1.0f), scale);
        int64_t o = i;
        if (part >= 0) {
            const int64_t r = i / cols, c = i % cols;
            o = ((r / 16) * 32 + part * 16 + (r % 16)) * cols + c;
        }
        dst[o] = f2bf(v);
    }
}

void init_weights(__nv_bfloat16* dst, uint64_t seed, uint64_t tensor_id, int64_t rows, int64_t cols,
                  float scale, int interleave_part, cudaStream_t stream) {
    init_weights_kernel<<<kNumSMs * 16, 256, 0, stream>>>(dst, seed, tensor_id, rows, cols, scale,
                                                          interleave_part);
}

__global__ void fill_bf16_kernel(__nv_bfloat16* dst, int64_t n, float v) {
    for (int64_t i = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; i < n;
         i += int64_t(gridDim.x) * blockDim.x)
        dst[i] = f2bf(v);
}
void fill_bf16(__nv_bfloat16* dst, int64_t n, float v, cudaStream_t stream) {
    fill_bf16_kernel<<<kNumSMs, 256, 0, stream>>>(dst, n, v);
}

// ---------------------------------------------------------- embedding ----
__global__ void embed_kernel(const __nv_bfloat16* __restrict__ emb, const int32_t* __restrict__ tok,
                             int d, __nv_bfloat16* __restrict__ x) {
    pdl_launch_dependents();
    pdl_wait();
    const int t = blockIdx.x;
    const uint4* src = reinterpret_cast<const uint4*>(emb + size_t(tok[t]) * d);
    uint4* dst = reinterpret_cast<uint4*>(x + size_t(t) * d);
    for (int i = threadIdx.x; i < d / 8; i += blockDim.x) dst[i] = src[i];
}
void embed_rows(const __nv_bfloat16* emb, const int32_t* tokens, int T, int d, __nv_bfloat16* x,
                cudaStream_t stream) {
    if (T > 0) launch_pdl(embed_kernel, dim3(T), dim3(128), 0, stream, emb, tokens, d, x);
}

// ------------------------------------------------------------ RMSNorm ----
// One CTA per row; d/8 16-byte vectors, at most 8 per thread kept in registers.
// Sum of 8 consecutive plane values (plane order) at element offset e; the loads of four planes
// are in flight at a time.
DS_DEVICE void sum_planes8(const Planes& pl, size_t e, float* acc) {
#pragma unroll
    for (int j = 0; j < 8; ++j) acc[j] = 0.f;
    for (int k0 = 0; k0 < pl.n; k0 += 4) {
        float4 a[4][2];
#pragma unroll
        for (int k = 0; k < 4; ++k)
            if (k0 + k < pl.n) {
                const float4* pk = reinterpret_cast<const float4*>(pl.p + (k0 + k) * pl.stride + e);
                a[k][0] = __ldcg(pk);
                a[k][1] = __ldcg(pk + 1);
            }
#pragma unroll
        for (int k = 0; k < 4; ++k)
            if (k0 + k < pl.n) {
                acc[0] += a[k][0].x; acc[1] += a[k][0].y; acc[2] += a[k][0].z; acc[3] += a[k][0].w;
                acc[4] += a[k][1].x; acc[5] += a[k][1].y; acc[6] += a[k][1].z; acc[7] += a[k][1].w;
            }
    }
}

template <int VPT>
__global__ void __launch_bounds__(512) rmsnorm_kernel(const __nv_bfloat16* __restrict__ x, const int32_t* __restrict__ rows,
                               int d, const __nv_bfloat16* __restrict__ g, float eps,
                               __nv_bfloat16* __restrict__ y, Planes pl) {
    pdl_launch_dependents();
    const int nv = d / 8;
    uint4 gq[VPT];  // gains: weights written at init, so loaded before the dependency wait
    if (y != nullptr) {
#pragma unroll
        for (int k = 0; k < VPT; ++k) {
            const int idx = threadIdx.x + k * blockDim.x;
            if (idx < nv) gq[k] = reinterpret_cast<const uint4*>(g)[idx];
        }
    }
    pdl_wait();
    const int i = blockIdx.x;
    const int src_row = rows ? rows[i] : i;
    const uint4* xr = reinterpret_cast<const uint4*>(x + size_t(src_row) * d);
    float v[VPT][8];
    float ss = 0.f;
#pragma unroll
    for (int k = 0; k < VPT; ++k) {
        const int idx = threadIdx.x + k * blockDim.x;
        if (idx < nv) {
            unpack8(xr[idx], v[k]);
            if (pl.n > 0) {  // deferred residual epilogue: x = bf16(x + bf16(acc))
                float acc[8];
                sum_planes8(pl, size_t(src_row) * d + idx * 8, acc);
#pragma unroll
                for (int j = 0; j < 8; ++j) v[k][j] = round_bf(v[k][j] + round_bf(acc[j]));
                reinterpret_cast<uint4*>(const_cast<__nv_bfloat16*>(x) + size_t(src_row) * d)[idx] = pack8(v[k]);
            }
#pragma unroll
            for (int j = 0; j < 8; ++j) ss += v[k][j] * v[k][j];
        }
    }
    if (y == nullptr) return;
    __shared__ float red[32];
    ss = warp_sum(ss);
    if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = ss;
    __syncthreads();
    if (threadIdx.x < 32) {
        float t = threadIdx.x < (blockDim.x >> 5) ? red[threadIdx.x] : 0.f;
        t = warp_sum(t);
        if (threadIdx.x == 0) red[0] = t;
    }
    __syncthreads();
    const float r = 1.0f / sqrtf(red[0] / float(d) + eps);
    uint4* yr = reinterpret_cast<uint4*>(y + size_t(i) * d);
#pragma unroll
    for (int k = 0; k < VPT; ++k) {
        const int idx = threadIdx.x + k * blockDim.x;
        if (idx < nv) {
            float gv[8], o[8];
            unpack8(gq[k], gv);
#pragma unroll
            for (int j = 0; j < 8; ++j) o[j] = gv[j] * round_bf(v[k][j] * r);
            yr[idx] = pack8(o);
        }
    }
}

void rmsnorm_rows(const __nv_bfloat16* x, const int32_t* rows, int n_rows, int d,
                  const __nv_bfloat16* g, float eps, __nv_bfloat16* y, cudaStream_t stream,
                  const Planes& pending) {
    if (n_rows <= 0) return;
    // one 16-byte vector per thread (d <= 4096) so every load of the row is in flight at once
    const int nv = d / 8;
    const int threads = std::min(512, std::max(32, (nv + 31) / 32 * 32));
    if (nv <= threads)
        launch_pdl(rmsnorm_kernel<1>, dim3(n_rows), dim3(threads), 0, stream, x, rows, d, g, eps, y, pending);
    else if (nv <= 4 * threads)
        launch_pdl(rmsnorm_kernel<4>, dim3(n_rows), dim3(threads), 0, stream, x, rows, d, g, eps, y, pending);
    else
        launch_pdl(rmsnorm_kernel<8>, dim3(n_rows), dim3(threads), 0, stream, x, rows, d, g, eps, y, pending);
}

// ------------------------------------------------- RoPE + KV append ----
__global__ void __launch_bounds__(512) rope_kv_kernel(const __nv_bfloat16* __restrict__ qkv, int n_h, int n_kv, int dh,
                               const int32_t* __restrict__ row_pos,
                               const int32_t* __restrict__ row_page, const float* __restrict__ rc,
                               const float* __restrict__ rs, KvLayout kv, int layer,
                               __nv_bfloat16* __restrict__ q_out, Planes pl) {
    pdl_launch_dependents();
    pdl_wait();
    const int t = blockIdx.x;
    const int pos = row_pos[t];
    const int half = dh / 2;
    // RowNorm scale of the row (q/k/v GEMM of the un-normalised x, planes deferred), published by
    // the GEMM; independent of the plane loads, so both are in flight together
    const float sc = (pl.n > 0 && pl.rs) ? __ldcg(pl.rs + t) : 1.f;
    const int width = (n_h + 2 * n_kv) * dh;
    const __nv_bfloat16* src = qkv + size_t(t) * width;
    const float* c = rc + size_t(pos) * half;
    const float* s = rs + size_t(pos) * half;
    const size_t page_base = size_t(row_page[t]) * kv.page_elems;
    const int slot = pos & 255;
    // rotated q and k: 8 consecutive rotary pairs per work item (16-byte accesses); then the v
    // vectors, 16 B per item. One flat index space so all of a row's loads are in flight together.
    const int n_rot = (n_h + n_kv) * (half / 8);
    const int nv = n_kv * dh / 8;
    for (int w = threadIdx.x; w < n_rot + nv; w += blockDim.x) {
        if (w >= n_rot) {
            const int kh = ((w - n_rot) * 8) / dh, i = ((w - n_rot) * 8) % dh;
            uint4 val;
            if (pl.n > 0) {
                float a[8];
                sum_planes8(pl, size_t(t) * width + (n_h + n_kv) * dh + kh * dh + i, a);
#pragma unroll
                for (int j = 0; j < 8; ++j) a[j] *= sc;
                val = pack8(a);
            } else {
                val = *reinterpret_cast<const uint4*>(src + (n_h + n_kv) * dh + kh * dh + i);
            }
            __nv_bfloat16* dv = kv.pool + page_base + ((size_t(layer) * 2 + 1) * n_kv + kh) * 256 * dh +
                                size_t(slot) * dh + i;
            *reinterpret_cast<uint4*>(dv) = val;
            continue;
        }
        const int head = w / (half / 8), i = (w % (half / 8)) * 8;
        float x1[8], x2[8], o1[8], o2[8];
        if (pl.n > 0) {  // deferred GEMM epilogue: bf16(sum of planes)
            sum_planes8(pl, size_t(t) * width + head * dh + i, x1);
            sum_planes8(pl, size_t(t) * width + head * dh + i + half, x2);
#pragma unroll
            for (int j = 0; j < 8; ++j) {
                x1[j] = round_bf(x1[j] * sc);
                x2[j] = round_bf(x2[j] * sc);
            }
        } else {
            unpack8(*reinterpret_cast<const uint4*>(src + head * dh + i), x1);
            unpack8(*reinterpret_cast<const uint4*>(src + head * dh + i + half), x2);
        }
        const float4 c0 = *reinterpret_cast<const float4*>(c + i), c1 = *reinterpret_cast<const float4*>(c + i + 4);
        const float4 s0 = *reinterpret_cast<const float4*>(s + i), s1 = *reinterpret_cast<const float4*>(s + i + 4);
        const float cc[8] = {c0.x, c0.y, c0.z, c0.w, c1.x, c1.y, c1.z, c1.w};
        const float ss[8] = {s0.x, s0.y, s0.z, s0.w, s1.x, s1.y, s1.z, s1.w};
#pragma unroll
        for (int j = 0; j < 8; ++j) {
            // explicit _rn ops: no FMA contraction, bit-identical to the CPU oracle
            o1[j] = __fsub_rn(__fmul_rn(x1[j], cc[j]), __fmul_rn(x2[j], ss[j]));
            o2[j] = __fadd_rn(__fmul_rn(x2[j], cc[j]), __fmul_rn(x1[j], ss[j]));
        }
        __nv_bfloat16* dst;
        if (head < n_h) {
            dst = q_out + size_t(t) * n_h * dh + head * dh;
        } else {
            dst = kv.pool + page_base + ((size_t(layer) * 2 + 0) * n_kv + (head - n_h)) * 256 * dh +
                  size_t(slot) * dh;
        }
        *reinterpret_cast<uint4*>(dst + i) = pack8(o1);
        *reinterpret_cast<uint4*>(dst + i + half) = pack8(o2);
    }
}

void rope_kv_append(const __nv_bfloat16* qkv, int T, int n_h, int n_kv, int d_head,
                    const int32_t* row_pos, const int32_t* row_page, const float* rope_cos,
                    const float* rope_sin, const KvLayout& kv, int layer, __nv_bfloat16* q_out,
                    cudaStream_t stream, const Planes& planes) {
    // one rotary 8-pair group or one v vector per thread: all loads of the row in flight
    const int work = (n_h + n_kv) * (d_head / 16) + n_kv * d_head / 8;
    const int threads = std::min(512, (work + 31) / 32 * 32);
    if (T > 0)
        launch_pdl(rope_kv_kernel, dim3(T), dim3(threads), 0, stream, qkv, n_h, n_kv, d_head, row_pos,
                   row_page, rope_cos, rope_sin, kv, layer, q_out, planes);
}

// ------------------------------------------------------------- argmax ----
__global__ void argmax_kernel(const float* __restrict__ logits, int V, int32_t* __restrict__ ids) {
    pdl_launch_dependents();
    pdl_wait();
    const float* row = logits + size_t(blockIdx.x) * V;
    float best = -INFINITY;
    int bi = 0x7fffffff;
    const int nv = V / 4;
    for (int i = threadIdx.x; i < nv; i += blockDim.x) {
        const float4 v = reinterpret_cast<const float4*>(row)[i];
        if (v.x > best) { best = v.x; bi = 4 * i; }
        if (v.y > best) { best = v.y; bi = 4 * i + 1; }
        if (v.z > best) { best = v.z; bi = 4 * i + 2; }
        if (v.w > best) { best = v.w; bi = 4 * i + 3; }
    }
    for (int i = nv * 4 + threadIdx.x; i < V; i += blockDim.x)
        if (row[i] > best) { best = row[i]; bi = i; }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
        const float ob = __shfl_xor_sync(0xffffffffu, best, o);
        const int oi = __shfl_xor_sync(0xffffffffu, bi, o);
        if (ob > best || (ob == best && oi < bi)) { best = ob; bi = oi; }
    }
    __shared__ float sb[32];
    __shared__ int si[32];
    if ((threadIdx.x & 31) == 0) { sb[threadIdx.x >> 5] = best; si[threadIdx.x >> 5] = bi; }
    __syncthreads();
    if (threadIdx.x < 32) {
        const int nw = blockDim.x >> 5;
        best = threadIdx.x < nw ? sb[threadIdx.x] : -INFINITY;
        bi = threadIdx.x < nw ? si[threadIdx.x] : 0x7fffffff;
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) {
            const float ob = __shfl_xor_sync(0xffffffffu, best, o);
            const int oi = __shfl_xor_sync(0xffffffffu, bi, o);
            if (ob > best || (ob == best && oi < bi)) { best = ob; bi = oi; }
        }
        if (threadIdx.x == 0) ids[blockIdx.x] = bi < V ? bi : 0;  // all-NaN row: stay in range
    }
}
void argmax_rows(const float* logits, int R, int V, int32_t* ids, cudaStream_t stream) {
    if (R > 0) launch_pdl(argmax_kernel, dim3(R), dim3(512), 0, stream, logits, V, ids);
}

__global__ void scatter_tokens_kernel(const int32_t* ids, const int32_t* req, int R, int32_t* last) {
    pdl_launch_dependents();
    pdl_wait();
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i < R) last[req[i]] = ids[i];
}
void scatter_tokens(const int32_t* ids, const int32_t* req, int R, int32_t* last_token,
                    cudaStream_t stream) {
    if (R > 0) launch_pdl(scatter_tokens_kernel, dim3((R + 255) / 256), dim3(256), 0, stream, ids, req, R, last_token);
}

__global__ void resolve_tokens_kernel(const int32_t* prompt_tok, const int32_t* row_req,
                                      const int32_t* last, int T, int32_t* tokens) {
    pdl_launch_dependents();
    pdl_wait();
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i < T) tokens[i] = prompt_tok[i] >= 0 ? prompt_tok[i] : last[row_req[i]];
}
void resolve_tokens(const int32_t* prompt_tok, const int32_t* row_req, const int32_t* last_token,
                    int T, int32_t* tokens, cudaStream_t stream) {
    if (T > 0)
        launch_pdl(resolve_tokens_kernel, dim3((T + 255) / 256), dim3(256), 0, stream, prompt_tok, row_req, last_token, T, tokens);
}

}  // namespace ds

namespace ds {
void preload_elementwise() {
    cudaFuncAttributes a;
    cudaFuncGetAttributes(&a, init_weights_kernel);
    cudaFuncGetAttributes(&a, fill_bf16_kernel);
    cudaFuncGetAttributes(&a, embed_kernel);
    cudaFuncGetAttributes(&a, rmsnorm_kernel<1>);
    cudaFuncGetAttributes(&a, rmsnorm_kernel<4>);
    cudaFuncGetAttributes(&a, rmsnorm_kernel<8>);
    cudaFuncGetAttributes(&a, rope_kv_kernel);
    cudaFuncGetAttributes(&a, argmax_kernel);
    cudaFuncGetAttributes(&a, scatter_tokens_kernel);
    cudaFuncGetAttributes(&a, resolve_tokens_kernel);
}
}  // namespace ds
