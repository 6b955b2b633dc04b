// Weight-streaming bf16 GEMM on 5th-generation tensor cores (tcgen05 + TMEM + TMA).
//
//   out[t, n] = epilogue( sum_k X[t, k] * W[n, k] )        X: [T, K], W: [N, K], both K-major
//
// Orientation: the weight matrix is the UMMA "A" operand (M = 128 output features per tile)
// and the stage's token rows are the "B" operand (N = up to 256 tokens per instruction, two
// instructions side by side for up to 512 tokens). A decode/prefill stage step has T = rows of
// the circuit (eff_batch, reference sim.cpp:406) which is small and ragged, so each CTA streams
// a 128-row weight panel from HBM exactly once per token block while the activations (tiny,
// L2-resident) are re-read. The fp32 accumulator lives in TMEM (lanes = features, columns =
// tokens); the epilogue warps drain it with tcgen05.ld and apply the fused epilogue.
//
// Warp roles (256 threads): w0 TMA producer, w1 MMA issuer, w2 TMEM allocator, w4..w7 epilogue.
// Work units = (token block, 128-feature tile, K split); persistent CTAs loop over units.
#include <cuda.h>

#include "common.cuh"
#include "kernels.h"

namespace ds {

constexpr int kBM = 128;   // weight rows per tile (UMMA M)
constexpr int kBK = 64;    // K elements per stage = one 128-byte swizzle row
constexpr int kMaxTB = 512;  // tokens per block (TMEM columns)
constexpr int kGemmThreads = 256;
constexpr int kSmemBudget = 200 * 1024;

struct GemmParams {
    int T, N, K;
    int k_splits;
    int t_blocks, m_tiles;
    int tb;        // tokens per block (<= 512)
    int bbox;      // TMA box rows for X (<= 256)
    int b_loads;   // X boxes per stage
    int stages;
    uint32_t tmem_cols;
    int epi;
    __nv_bfloat16* out_bf16;
    const __nv_bfloat16* resid;
    float* out_f32;  // EPI_F32 output or split-K workspace [k_splits][T][N]
};

__global__ void __launch_bounds__(kGemmThreads, 1)
gemm_tc_kernel(const __grid_constant__ CUtensorMap tmap_w, const __grid_constant__ CUtensorMap tmap_x,
               const GemmParams p) {
    extern __shared__ __align__(1024) uint8_t smem_raw[];
    // 1024-byte alignment for SWIZZLE_128B tiles.
    uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) &
                                               ~uintptr_t(1023));
    const int a_bytes = kBM * kBK * 2;
    const int b_bytes = p.b_loads * p.bbox * kBK * 2;
    const int stage_bytes = a_bytes + b_bytes;
    uint64_t* full_bar = reinterpret_cast<uint64_t*>(smem + p.stages * stage_bytes);
    uint64_t* empty_bar = full_bar + p.stages;
    uint64_t* tfull_bar = empty_bar + p.stages;
    uint64_t* tempty_bar = tfull_bar + 1;
    uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(tempty_bar + 1);

    const int warp = threadIdx.x >> 5;
    const int lane = threadIdx.x & 31;

    if (warp == 0 && lane == 0) {
        tma_prefetch_desc(&tmap_w);
        tma_prefetch_desc(&tmap_x);
        for (int s = 0; s < p.stages; ++s) {
            mbar_init(&full_bar[s], 1);
            mbar_init(&empty_bar[s], 1);
        }
        mbar_init(tfull_bar, 1);
        mbar_init(tempty_bar, 4);
        fence_mbar_init();
    }
    if (warp == 2) tmem_alloc(tmem_slot, p.tmem_cols);
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tmem_base = *tmem_slot;

    const int total_kb = p.K / kBK;
    const int units = p.t_blocks * p.m_tiles * p.k_splits;

    pdl_launch_dependents();  // the next kernel may start its prologue on SMs we free

    if (warp == 0) {
        if (elect_one()) {
            const uint64_t pol_w = policy_evict_first();
            // The weights do not depend on the previous kernel: issue the first `stages` weight
            // tiles before waiting for it (programmatic dependent launch), the activations after.
            int pre = 0;
            for (int u = blockIdx.x; u < units && pre < p.stages; u += gridDim.x) {
                const int ks = u % p.k_splits;
                const int mt = (u / p.k_splits) % p.m_tiles;
                const int kb0 = ks * total_kb / p.k_splits;
                const int kb1 = (ks + 1) * total_kb / p.k_splits;
                for (int kb = kb0; kb < kb1 && pre < p.stages; ++kb, ++pre) {
                    uint8_t* sa = smem + pre * stage_bytes;
                    mbar_arrive_expect_tx(&full_bar[pre], stage_bytes);
                    tma_load_2d_hint(sa, &tmap_w, &full_bar[pre], kb * kBK, mt * kBM, pol_w);
                }
            }
            pdl_wait();
            int it = 0;
            for (int u = blockIdx.x; u < units; u += gridDim.x) {
                const int ks = u % p.k_splits;
                const int mt = (u / p.k_splits) % p.m_tiles;
                const int tbk = u / (p.k_splits * p.m_tiles);
                const int kb0 = ks * total_kb / p.k_splits;
                const int kb1 = (ks + 1) * total_kb / p.k_splits;
                for (int kb = kb0; kb < kb1; ++kb, ++it) {
                    const int s = it % p.stages;
                    const uint32_t round = it / p.stages;
                    uint8_t* sa = smem + s * stage_bytes;
                    uint8_t* sb = sa + a_bytes;
                    if (it >= pre) {
                        mbar_wait(&empty_bar[s], (round & 1) ^ 1);
                        mbar_arrive_expect_tx(&full_bar[s], stage_bytes);
                        tma_load_2d_hint(sa, &tmap_w, &full_bar[s], kb * kBK, mt * kBM, pol_w);
                    }
                    for (int j = 0; j < p.b_loads; ++j)
                        tma_load_2d(sb + j * p.bbox * kBK * 2, &tmap_x, &full_bar[s], kb * kBK,
                                    tbk * p.tb + j * p.bbox);
                }
            }
        }
    } else if (warp == 1) {
        int it = 0;
        int uc = 0;
        for (int u = blockIdx.x; u < units; u += gridDim.x, ++uc) {
            const int ks = u % p.k_splits;
            const int tbk = u / (p.k_splits * p.m_tiles);
            const int kb0 = ks * total_kb / p.k_splits;
            const int kb1 = (ks + 1) * total_kb / p.k_splits;
            const int t_here = min(p.tb, p.T - tbk * p.tb);
            mbar_wait(tempty_bar, (uc & 1) ^ 1);
            tc_fence_after();
            for (int kb = kb0; kb < kb1; ++kb, ++it) {
                const int s = it % p.stages;
                const uint32_t round = it / p.stages;
                mbar_wait(&full_bar[s], round & 1);
                tc_fence_after();
                if (elect_one()) {
                    const uint32_t sa = smem_u32(smem + s * stage_bytes);
                    const uint32_t sb = sa + a_bytes;
#pragma unroll
                    for (int c = 0; c < 2; ++c) {
                        const int n_c = min(256, t_here - 256 * c);
                        if (n_c <= 0) break;
                        const int n_pad = (n_c + 15) & ~15;
                        const uint32_t idesc = umma_idesc_bf16(kBM, n_pad);
#pragma unroll
                        for (int k = 0; k < kBK / 16; ++k) {
                            const uint64_t ad = umma_sdesc_sw128(sa + k * 32);
                            const uint64_t bd = umma_sdesc_sw128(sb + c * 256 * 128 + k * 32);
                            umma_bf16(tmem_base + c * 256, ad, bd, idesc,
                                      (kb > kb0 || k > 0) ? 1u : 0u);
                        }
                    }
                    umma_commit(&empty_bar[s]);
                    if (kb == kb1 - 1) umma_commit(tfull_bar);
                }
                __syncwarp();
            }
        }
    } else if (warp >= 4) {
        pdl_wait();
        const int q = warp & 3;
        int uc = 0;
        for (int u = blockIdx.x; u < units; u += gridDim.x, ++uc) {
            const int ks = u % p.k_splits;
            const int mt = (u / p.k_splits) % p.m_tiles;
            const int tbk = u / (p.k_splits * p.m_tiles);
            const int t0 = tbk * p.tb;
            const int t_here = min(p.tb, p.T - t0);
            const int n = mt * kBM + q * 32 + lane;
            mbar_wait(tfull_bar, uc & 1);
            tc_fence_after();
            for (int c0 = 0; c0 < t_here; c0 += 16) {
                uint32_t r[16];
                tmem_ld16(tmem_base + (uint32_t(q * 32) << 16) + c0, r);
                tmem_ld_wait();
                const int tmax = min(16, t_here - c0);
                if (p.epi == EPI_BF16) {
                    for (int j = 0; j < tmax; ++j)
                        p.out_bf16[size_t(t0 + c0 + j) * p.N + n] = f2bf(__uint_as_float(r[j]));
                } else if (p.epi == EPI_RESID) {
                    for (int j = 0; j < tmax; ++j) {
                        const size_t o = size_t(t0 + c0 + j) * p.N + n;
                        const float y = bf2f(p.resid[o]) + round_bf(__uint_as_float(r[j]));
                        p.out_bf16[o] = f2bf(y);
                    }
                } else {
                    float* dst = p.out_f32 + (p.epi == EPI_PARTIAL ? size_t(ks) * p.T * p.N : 0);
                    for (int j = 0; j < tmax; ++j)
                        dst[size_t(t0 + c0 + j) * p.N + n] = __uint_as_float(r[j]);
                }
            }
            tc_fence_before();
            __syncwarp();
            if (lane == 0) mbar_arrive(tempty_bar);
        }
    }
    __syncthreads();
    if (warp == 2) {
        tc_fence_after();
        tmem_dealloc(tmem_base, p.tmem_cols);
    }
}

// Deterministic split-K reduction (splits summed in order) + the same epilogues.
__global__ void splitk_reduce_kernel(const float* __restrict__ ws, int splits, int T, int N, int epi,
                                     __nv_bfloat16* out_bf16, const __nv_bfloat16* resid,
                                     float* out_f32) {
    pdl_launch_dependents();
    pdl_wait();
    const size_t total = size_t(T) * N / 4;
    const size_t plane = size_t(T) * N;
    for (size_t i = blockIdx.x * size_t(blockDim.x) + threadIdx.x; i < total;
         i += size_t(gridDim.x) * blockDim.x) {
        float4 acc = reinterpret_cast<const float4*>(ws)[i];
        for (int s = 1; s < splits; ++s) {
            const float4 v = reinterpret_cast<const float4*>(ws + s * plane)[i];
            acc.x += v.x;
            acc.y += v.y;
            acc.z += v.z;
            acc.w += v.w;
        }
        const size_t o = i * 4;
        if (epi == EPI_F32) {
            reinterpret_cast<float4*>(out_f32)[i] = acc;
        } else {
            float a[4] = {acc.x, acc.y, acc.z, acc.w};
            if (epi == EPI_RESID) {
                const uint2 rv = *reinterpret_cast<const uint2*>(resid + o);
                const __nv_bfloat162* rh = reinterpret_cast<const __nv_bfloat162*>(&rv);
                const float2 r0 = __bfloat1622float2(rh[0]);
                const float2 r1 = __bfloat1622float2(rh[1]);
                a[0] = r0.x + round_bf(a[0]);
                a[1] = r0.y + round_bf(a[1]);
                a[2] = r1.x + round_bf(a[2]);
                a[3] = r1.y + round_bf(a[3]);
            }
            uint2 ov;
            ov.x = pack2(a[0], a[1]);
            ov.y = pack2(a[2], a[3]);
            *reinterpret_cast<uint2*>(out_bf16 + o) = ov;
        }
    }
}

// ------------------------------------------------------------------ host ----

using EncodeTiledFn = CUresult (*)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                                   const cuuint64_t*, const cuuint32_t*, const cuuint32_t*,
                                   CUtensorMapInterleave, CUtensorMapSwizzle,
                                   CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

static EncodeTiledFn get_encode_fn() {
    static EncodeTiledFn fn = nullptr;
    if (!fn) {
        cudaDriverEntryPointQueryResult q;
        void* p = nullptr;
        cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q);
        fn = reinterpret_cast<EncodeTiledFn>(p);
    }
    return fn;
}

int make_tmap_2d_bf16(void* tmap_out, const void* base, uint64_t rows, uint64_t cols,
                      uint32_t box_rows, uint32_t box_cols) {
    auto fn = get_encode_fn();
    if (!fn) return -1;
    CUtensorMap* m = reinterpret_cast<CUtensorMap*>(tmap_out);
    cuuint64_t dims[2] = {cols, rows};
    cuuint64_t strides[1] = {cols * 2};
    cuuint32_t box[2] = {box_cols, box_rows};
    cuuint32_t estr[2] = {1, 1};
    CUresult r = fn(m, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, const_cast<void*>(base), dims, strides,
                    box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                    CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    return r == CUDA_SUCCESS ? 0 : -2;
}

size_t gemm_workspace_floats(int T, int N, int k_splits) { return size_t(k_splits) * T * N; }

int gemm_pick_splits(int T, int N, int K) {
    const int tiles = ((T + kMaxTB - 1) / kMaxTB) * (N / kBM);
    const int kb = K / kBK;
    if (tiles >= kNumSMs / 2) return 1;
    int s = kNumSMs / tiles;
    s = min(s, 8);
    s = min(s, kb / 4);
    return max(s, 1);
}

int gemm_bf16(const GemmWeight& w, const __nv_bfloat16* x, int T, int epi, __nv_bfloat16* out_bf16,
              const __nv_bfloat16* resid, float* out_f32, float* workspace, size_t workspace_floats,
              int k_splits, cudaStream_t stream) {
    const int N = w.N, K = w.K;
    if (T <= 0) return 0;
    if (K % kBK != 0 || N % kBM != 0) return -3;
    GemmParams p{};
    p.T = T;
    p.N = N;
    p.K = K;
    p.t_blocks = (T + kMaxTB - 1) / kMaxTB;
    p.tb = T < kMaxTB ? T : kMaxTB;
    const int tb_pad = (p.tb + 15) & ~15;
    p.bbox = tb_pad < 256 ? tb_pad : 256;
    p.b_loads = (tb_pad + p.bbox - 1) / p.bbox;
    p.m_tiles = N / kBM;
    if (k_splits <= 0) k_splits = gemm_pick_splits(T, N, K);
    if (k_splits > 1 && (size_t(k_splits) * T * N > workspace_floats || workspace == nullptr))
        k_splits = 1;
    p.k_splits = k_splits;
    const int stage_bytes = kBM * kBK * 2 + p.b_loads * p.bbox * kBK * 2;
    p.stages = (kSmemBudget - 2048) / stage_bytes;
    if (p.stages > 8) p.stages = 8;
    if (p.stages < 2) return -4;
    uint32_t cols = 32;
    while (cols < uint32_t(tb_pad > 256 ? 512 : tb_pad)) cols <<= 1;
    p.tmem_cols = cols;
    if (k_splits > 1) {
        p.epi = EPI_PARTIAL;
        p.out_f32 = workspace;
    } else {
        p.epi = epi;
        p.out_bf16 = out_bf16;
        p.resid = resid;
        p.out_f32 = out_f32;
    }
    alignas(64) CUtensorMap tx;
    if (make_tmap_2d_bf16(&tx, x, T, K, p.bbox, kBK) != 0) return -5;
    const size_t smem = size_t(p.stages) * stage_bytes + 1024 + 256;
    static bool attr_set = false;
    if (!attr_set) {
        cudaFuncSetAttribute(gemm_tc_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                             kSmemBudget + 2048);
        attr_set = true;
    }
    const int units = p.t_blocks * p.m_tiles * p.k_splits;
    const int grid = units < kNumSMs ? units : kNumSMs;
    launch_pdl(gemm_tc_kernel, dim3(grid), dim3(kGemmThreads), smem, stream,
               *reinterpret_cast<const CUtensorMap*>(w.tmap), tx, p);
    if (k_splits > 1) {
        const size_t total4 = size_t(T) * N / 4;
        int blocks = int((total4 + 255) / 256);
        if (blocks > kNumSMs * 8) blocks = kNumSMs * 8;
        launch_pdl(splitk_reduce_kernel, dim3(blocks), dim3(256), 0, stream, (const float*)workspace,
                   k_splits, T, N, epi, out_bf16, resid, out_f32);
    }
    return cudaPeekAtLastError() == cudaSuccess ? 0 : -6;
}

int gemm_weight_init(GemmWeight* w, const __nv_bfloat16* data, int N, int K) {
    w->data = data;
    w->N = N;
    w->K = K;
    return make_tmap_2d_bf16(w->tmap, data, N, K, kBM, kBK);
}

}  // namespace ds

namespace ds {
// Forces the module holding these kernels to load now (lazy loading would otherwise load it at
// the first launch, which can wait on in-flight work such as a spinning NCCL receive).
void preload_gemm() {
    cudaFuncAttributes a;
    cudaFuncGetAttributes(&a, gemm_tc_kernel);
    cudaFuncGetAttributes(&a, splitk_reduce_kernel);
    cudaFuncSetAttribute(gemm_tc_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, kSmemBudget + 2048);
}
}  // namespace ds
