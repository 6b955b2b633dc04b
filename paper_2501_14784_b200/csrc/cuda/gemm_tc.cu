// Weight-streaming bf16 GEMM on 5th-generation tensor cores (tcgen05 + TMEM + TMA).
//
//   out[t, n] = epilogue( sum_k X[t, k] * W[n, k] )        X: [T, K], W: [N, K], both K-major
//
// Orientation: the weight matrix is the UMMA "A" operand (M = 128 output features per CTA tile)
// and the stage step's token rows are the "B" operand (N <= 256 tokens per instruction, two
// instructions side by side for <= 512 tokens per token block). A stage step has T = eff_batch
// rows (reference sim.cpp:406): small and ragged, so weights are streamed from HBM exactly once
// per token block, the fp32 accumulator lives in TMEM (lanes = features, columns = tokens).
//
// * 2-CTA clusters: the two CTAs of a cluster own adjacent 128-feature tiles and the same token
//   block; each loads half of the activation tile and multicasts it to both (TMA .multicast), so
//   the per-SM activation traffic from L2 is halved. Each CTA's MMA releases a stage in both
//   CTAs (tcgen05.commit .multicast::cluster).
// * Work units = (cluster tile, K split), handed to clusters round-robin (persistent CTAs). Wide
//   GEMMs (>= one wave of cluster tiles) run unsplit; narrow ones (q/k/v, o, down at 8B) split K
//   so every SM streams weights, parking fp32 partials that a PDL-chained reduction kernel sums
//   in split order (deterministic) with the same fused epilogue. (An in-kernel stream-K fixup was
//   measured slower here: its contributors idle while the tile's last partial lands.)
// * TMEM holds two accumulators when the token block fits 256 columns, so a unit's epilogue
//   overlaps the next unit's MMAs.
// * Epilogue: tcgen05.ld -> shared-memory transpose -> 16-byte coalesced stores, fused
//   bf16 / residual-add (x = bf16(x + bf16(acc))) / fp32 (logits, split partials).
// * Programmatic dependent launch: the first weight tiles are fetched before waiting on the
//   previous kernel; the activations after.
//
// Warp roles (256 threads): w0 TMA producer, w1 MMA issuer, w2 TMEM allocator, w4..w7 epilogue.
#include <cuda.h>

#include <algorithm>
#include <cstdlib>

#include "common.cuh"
#include "kernels.h"

namespace ds {

constexpr int kBM = 128;      // weight rows per CTA tile (UMMA M)
constexpr int kBK = 64;       // K elements per stage = one 128-byte swizzle row
constexpr int kMaxTB = 512;   // tokens per block (TMEM columns)
constexpr int kGemmThreads = 256;
constexpr int kSmemBudget = 222 * 1024;
constexpr int kStageStride = 36;  // floats per row of the epilogue transpose buffer
constexpr size_t kWorkspaceFloats = size_t(16) << 20;  // split-K partials

struct GemmParams {
    int T, N, K;
    int m_tiles;  // N / 128
    int t_blocks;
    int tb;       // tokens per block (<= 512)
    int tb_pad;   // tb rounded up to 16
    int brows;    // activation rows each CTA of the cluster loads per stage (tb_pad / CN)
    int stages;
    int n_acc;    // TMEM accumulators
    int KB;       // k-blocks per tile
    int splits;   // K splits per tile
    int n_clusters;
    int units;    // cluster tiles x splits
    int epi;
    __nv_bfloat16* out_bf16;
    const __nv_bfloat16* resid;
    float* out_f32;
    float* partial;  // [splits][T][N] fp32 when splits > 1
    unsigned long long* trace;  // optional per-CTA phase timestamps (gemm_set_trace)
};

DS_DEVICE unsigned long long gtime() {
    unsigned long long t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    return t;
}
#define GEMM_TRACE(k)                                             \
    do {                                                          \
        if (p.trace) p.trace[blockIdx.x * 8 + (k)] = gtime();    \
    } while (0)

static unsigned long long* g_gemm_trace = nullptr;
void gemm_set_trace(unsigned long long* buf) { g_gemm_trace = buf; }

DS_DEVICE uint32_t cluster_rank() {
    uint32_t r;
    asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
    return r;
}
DS_DEVICE void cluster_sync() {
    asm volatile("barrier.cluster.arrive.release.aligned;\nbarrier.cluster.wait.acquire.aligned;" ::: "memory");
}
DS_DEVICE void tma_load_2d_mc(void* smem_dst, const void* tmap, uint64_t* bar, int c0, int c1,
                              uint16_t mask) {
    asm volatile(
        "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes.multicast::cluster"
        " [%0], [%1, {%3, %4}], [%2], %5;" ::"r"(smem_u32(smem_dst)),
        "l"(reinterpret_cast<uint64_t>(tmap)), "r"(smem_u32(bar)), "r"(c0), "r"(c1), "h"(mask)
        : "memory");
}
DS_DEVICE void umma_commit_mc(uint64_t* bar, uint16_t mask) {
    asm volatile(
        "tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64"
        " [%0], %1;" ::"r"(smem_u32(bar)),
        "h"(mask)
        : "memory");
}

// A unit: cluster tile ut (token block x feature pair) and its K range [kb0, kb1).
struct Unit {
    int ut, split, kb0, kb1;
};
DS_DEVICE Unit unit_of(const GemmParams& p, int u) {
    Unit x;
    x.ut = u / p.splits;
    x.split = u % p.splits;
    x.kb0 = x.split * p.KB / p.splits;
    x.kb1 = (x.split + 1) * p.KB / p.splits;
    return x;
}

// Applies the epilogue to 16 consecutive token columns of one 32-feature slice held as vals[16]
// (this thread's feature, columns c0..c0+15), through a per-warp transpose buffer.
DS_DEVICE void epilogue16(const GemmParams& p, int epi, float* out_f32, float* stage,
                          const float* vals, int lane, int t0, int c0, int t_here, int f_base) {
#pragma unroll
    for (int j = 0; j < 16; ++j) stage[j * kStageStride + lane] = vals[j];
    __syncwarp();
    const int row = lane >> 1, half = lane & 1;
    if (c0 + row < t_here) {
        const int t = t0 + c0 + row;
        const int f0 = f_base + half * 16;
        const float4* src = reinterpret_cast<const float4*>(stage + row * kStageStride + half * 16);
        float v[16];
#pragma unroll
        for (int i = 0; i < 4; ++i) {
            const float4 x = src[i];
            v[4 * i] = x.x;
            v[4 * i + 1] = x.y;
            v[4 * i + 2] = x.z;
            v[4 * i + 3] = x.w;
        }
        const size_t o = size_t(t) * p.N + f0;
        if (epi == EPI_F32) {
            float4* dst = reinterpret_cast<float4*>(out_f32 + o);
#pragma unroll
            for (int i = 0; i < 4; ++i) dst[i] = make_float4(v[4 * i], v[4 * i + 1], v[4 * i + 2], v[4 * i + 3]);
        } else {
            if (epi == EPI_RESID) {
                float r[16];
                unpack8(reinterpret_cast<const uint4*>(p.resid + o)[0], r);
                unpack8(reinterpret_cast<const uint4*>(p.resid + o)[1], r + 8);
#pragma unroll
                for (int j = 0; j < 16; ++j) v[j] = r[j] + round_bf(v[j]);
            }
            uint4* dst = reinterpret_cast<uint4*>(p.out_bf16 + o);
            dst[0] = pack8(v);
            dst[1] = pack8(v + 8);
        }
    }
    __syncwarp();
}

template <int CN>
__global__ void __launch_bounds__(kGemmThreads, 1)
gemm_tc_kernel(const __grid_constant__ CUtensorMap tmap_w, const __grid_constant__ CUtensorMap tmap_x,
               const GemmParams p) {
    extern __shared__ __align__(1024) uint8_t smem_raw[];
    uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) &
                                               ~uintptr_t(1023));
    const int a_bytes = kBM * kBK * 2;
    const int b_bytes = p.tb_pad * kBK * 2;
    const int stage_bytes = a_bytes + b_bytes;
    float* ep_stage = reinterpret_cast<float*>(smem + p.stages * stage_bytes);  // 4 x 16 x 36 floats
    uint64_t* full_bar = reinterpret_cast<uint64_t*>(ep_stage + 4 * 16 * kStageStride);
    uint64_t* empty_bar = full_bar + p.stages;
    uint64_t* tfull_bar = empty_bar + p.stages;  // [2]
    uint64_t* tempty_bar = tfull_bar + 2;        // [2]
    uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(tempty_bar + 2);

    const int warp = threadIdx.x >> 5;
    const int lane = threadIdx.x & 31;
    const uint32_t rank = CN > 1 ? cluster_rank() : 0;
    const int cluster = blockIdx.x / CN;

    if (warp == 0 && lane == 0) {
        tma_prefetch_desc(&tmap_w);
        tma_prefetch_desc(&tmap_x);
        for (int s = 0; s < p.stages; ++s) {
            mbar_init(&full_bar[s], 1);
            mbar_init(&empty_bar[s], CN);
        }
        for (int a = 0; a < 2; ++a) {
            mbar_init(&tfull_bar[a], 1);
            mbar_init(&tempty_bar[a], 4);
        }
        fence_mbar_init();
    }
    if (warp == 2) tmem_alloc(tmem_slot, 512);
    tc_fence_before();
    __syncthreads();
    if (CN > 1) cluster_sync();  // remote barriers initialised before any multicast lands
    tc_fence_after();
    const uint32_t tmem_base = *tmem_slot;
    if (threadIdx.x == 0) GEMM_TRACE(0);
    pdl_launch_dependents();

    const int cl_tiles = p.m_tiles / CN;

    if (warp == 0) {
        if (elect_one()) {
            const uint64_t pol_w = policy_evict_first();
            const uint16_t mask = (1u << CN) - 1;
            // weights first (independent of the previous kernel), activations after pdl_wait
            int pre = 0;
            for (int u = cluster; u < p.units && pre < p.stages; u += p.n_clusters) {
                const Unit w = unit_of(p, u);
                const int mt = (w.ut % cl_tiles) * CN + int(rank);
                for (int kb = w.kb0; kb < w.kb1 && pre < p.stages; ++kb, ++pre) {
                    mbar_arrive_expect_tx(&full_bar[pre], stage_bytes);
                    tma_load_2d_hint(smem + pre * stage_bytes, &tmap_w, &full_bar[pre], kb * kBK,
                                     mt * kBM, pol_w);
                }
            }
            pdl_wait();
            int i = 0;
            for (int u = cluster; u < p.units; u += p.n_clusters) {
                const Unit w = unit_of(p, u);
                const int tbk = w.ut / cl_tiles;
                const int mt = (w.ut % cl_tiles) * CN + int(rank);
                for (int kb = w.kb0; kb < w.kb1; ++kb, ++i) {
                    const int s = i % p.stages;
                    const uint32_t round = i / p.stages;
                    uint8_t* sa = smem + s * stage_bytes;
                    uint8_t* sb = sa + a_bytes;
                    if (i >= pre) {
                        mbar_wait(&empty_bar[s], (round & 1) ^ 1);
                        mbar_arrive_expect_tx(&full_bar[s], stage_bytes);
                        tma_load_2d_hint(sa, &tmap_w, &full_bar[s], kb * kBK, mt * kBM, pol_w);
                    }
                    if (CN > 1)
                        tma_load_2d_mc(sb + rank * p.brows * kBK * 2, &tmap_x, &full_bar[s], kb * kBK,
                                       tbk * p.tb + int(rank) * p.brows, mask);
                    else
                        tma_load_2d(sb, &tmap_x, &full_bar[s], kb * kBK, tbk * p.tb);
                }
            }
            GEMM_TRACE(1);
            // drain: every stage released by every CTA (no remote arrival after we exit)
            const int n = i;
            for (int k = (n > p.stages ? n - p.stages : 0); k < n; ++k)
                mbar_wait(&empty_bar[k % p.stages], (uint32_t(k / p.stages) & 1));
        }
    } else if (warp == 1) {
        int i = 0, seg = 0;
        for (int u = cluster; u < p.units; u += p.n_clusters, ++seg) {
            const Unit w = unit_of(p, u);
            const int tbk = w.ut / cl_tiles;
            const int t_here = min(p.tb, p.T - tbk * p.tb);
            const int a = seg % p.n_acc;
            const uint32_t acc = tmem_base + uint32_t(a * 256);
            mbar_wait(&tempty_bar[a], ((seg / p.n_acc) & 1) ^ 1);
            tc_fence_after();
            for (int kb = w.kb0; kb < w.kb1; ++kb, ++i) {
                const int s = i % p.stages;
                mbar_wait(&full_bar[s], (i / p.stages) & 1);
                tc_fence_after();
                if (elect_one()) {
                    const uint32_t sa = smem_u32(smem + s * stage_bytes);
                    const uint32_t sb = sa + a_bytes;
#pragma unroll
                    for (int c = 0; c < 2; ++c) {
                        const int n_c = min(256, t_here - 256 * c);
                        if (n_c <= 0) break;
                        const uint32_t idesc = umma_idesc_bf16(kBM, (n_c + 15) & ~15);
#pragma unroll
                        for (int k = 0; k < kBK / 16; ++k)
                            umma_bf16(acc + c * 256, umma_sdesc_sw128(sa + k * 32),
                                      umma_sdesc_sw128(sb + c * 256 * 128 + k * 32), idesc,
                                      (kb > w.kb0 || k > 0) ? 1u : 0u);
                    }
                    if (CN > 1)
                        umma_commit_mc(&empty_bar[s], (1u << CN) - 1);
                    else
                        umma_commit(&empty_bar[s]);
                    if (kb == w.kb1 - 1) umma_commit(&tfull_bar[a]);
                }
                __syncwarp();
            }
        }
        if (lane == 0) GEMM_TRACE(2);
    } else if (warp >= 4) {
        pdl_wait();
        const int q = warp & 3;
        float* stage = ep_stage + q * 16 * kStageStride;
        int seg = 0;
        for (int u = cluster; u < p.units; u += p.n_clusters, ++seg) {
            const Unit w = unit_of(p, u);
            const int tbk = w.ut / cl_tiles;
            const int mt = (w.ut % cl_tiles) * CN + int(rank);
            const int t0 = tbk * p.tb;
            const int t_here = min(p.tb, p.T - t0);
            const int a = seg % p.n_acc;
            const uint32_t acc = tmem_base + uint32_t(a * 256) + (uint32_t(q * 32) << 16);
            mbar_wait(&tfull_bar[a], (seg / p.n_acc) & 1);
            tc_fence_after();
            // unsplit: the fused epilogue; split: an fp32 partial into its split plane
            const int epi = p.splits > 1 ? EPI_F32 : p.epi;
            float* out_f32 = p.splits > 1 ? p.partial + size_t(w.split) * p.T * p.N : p.out_f32;
            for (int c0 = 0; c0 < t_here; c0 += 16) {
                uint32_t r[16];
                tmem_ld16(acc + c0, r);
                tmem_ld_wait();
                epilogue16(p, epi, out_f32, stage, reinterpret_cast<float*>(r), lane, t0, c0, t_here,
                           mt * kBM + q * 32);
            }
            tc_fence_before();
            __syncwarp();
            if (lane == 0) mbar_arrive(&tempty_bar[a]);
        }
        if (threadIdx.x == 128) GEMM_TRACE(3);
    }
    __syncthreads();
    if (CN > 1) cluster_sync();
    if (warp == 2) {
        tc_fence_after();
        tmem_dealloc(tmem_base, 512);
    }
}

// Split-K reduction: splits summed in order (deterministic) + the same epilogues.
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
        void* ptr = nullptr;
        cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &ptr, cudaEnableDefault, &q);
        fn = reinterpret_cast<EncodeTiledFn>(ptr);
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

size_t gemm_workspace_floats() { return kWorkspaceFloats; }

// launches issued by gemm_bf16 for this shape (1, or 2 with the split-K reduction)
int gemm_launch_count(int T, int N, int K);

static int pick_splits(int T, int N, int K, int cn, int n_clusters) {
    const int tiles = ((T + kMaxTB - 1) / kMaxTB) * (N / kBM / cn);
    if (tiles >= n_clusters) return 1;
    int s = n_clusters / tiles;
    s = std::min(s, 8);
    s = std::min(s, (K / kBK) / 4);
    while (s > 1 && size_t(s) * T * N > kWorkspaceFloats) --s;
    return std::max(s, 1);
}

static int pick_cn(int N) {
    static const int cn_env = getenv("DS_GEMM_CN") ? atoi(getenv("DS_GEMM_CN")) : 2;
    return (cn_env == 1 || (N / kBM) % 2 != 0) ? 1 : 2;
}

int gemm_launch_count(int T, int N, int K) {
    const int cn = pick_cn(N);
    return pick_splits(T, N, K, cn, kNumSMs / cn) > 1 ? 2 : 1;
}

int gemm_bf16(const GemmWeight& w, const __nv_bfloat16* x, int T, int epi, __nv_bfloat16* out_bf16,
              const __nv_bfloat16* resid, float* out_f32, float* workspace, size_t workspace_floats,
              int max_clusters, cudaStream_t stream) {
    const int N = w.N, K = w.K;
    if (T <= 0) return 0;
    int cn = pick_cn(N);
    if (K % kBK != 0 || N % kBM != 0) return -3;
    GemmParams p{};
    p.T = T;
    p.N = N;
    p.K = K;
    p.m_tiles = N / kBM;
    p.t_blocks = (T + kMaxTB - 1) / kMaxTB;
    p.tb = T < kMaxTB ? T : kMaxTB;
    p.tb_pad = (p.tb + 15) & ~15;
    if (cn == 1 && p.tb_pad > 256) cn = (p.m_tiles % 2 == 0) ? 2 : 1;  // TMA box rows <= 256
    if (cn == 1 && p.tb_pad > 256) return -9;
    p.brows = p.tb_pad / cn;
    p.KB = K / kBK;
    const int stage_bytes = kBM * kBK * 2 + p.tb_pad * kBK * 2;
    const int fixed = 4 * 16 * kStageStride * 4 + 256 + 1024;
    p.stages = (kSmemBudget - fixed) / stage_bytes;
    if (p.stages > 12) p.stages = 12;
    if (p.stages < 2) return -4;
    p.n_acc = p.tb_pad <= 256 ? 2 : 1;
    int nc = kNumSMs / cn;
    if (max_clusters > 0 && nc > max_clusters) nc = max_clusters;
    p.splits = pick_splits(T, N, K, cn, nc);
    if (p.splits > 1 && (!workspace || workspace_floats < size_t(p.splits) * T * N)) p.splits = 1;
    const int tiles = p.t_blocks * (p.m_tiles / cn);
    p.units = tiles * p.splits;
    p.n_clusters = std::min(nc, p.units);
    p.epi = epi;
    p.out_bf16 = out_bf16;
    p.resid = resid;
    p.out_f32 = out_f32;
    p.partial = workspace;
    p.trace = g_gemm_trace;
    alignas(64) CUtensorMap tx;
    if (make_tmap_2d_bf16(&tx, x, T, K, p.brows, kBK) != 0) return -5;
    const size_t smem = size_t(p.stages) * stage_bytes + fixed;
    cudaLaunchConfig_t cfg{};
    cfg.gridDim = dim3(p.n_clusters * cn);
    cfg.blockDim = dim3(kGemmThreads);
    cfg.dynamicSmemBytes = smem;
    cfg.stream = stream;
    cudaLaunchAttribute attr[2];
    attr[0].id = cudaLaunchAttributeClusterDimension;
    attr[0].val.clusterDim.x = cn;
    attr[0].val.clusterDim.y = 1;
    attr[0].val.clusterDim.z = 1;
    attr[1].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[1].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 2;
    const CUtensorMap& tw = *reinterpret_cast<const CUtensorMap*>(w.tmap);
    cudaError_t e = cn == 2 ? cudaLaunchKernelEx(&cfg, gemm_tc_kernel<2>, tw, tx, p)
                            : cudaLaunchKernelEx(&cfg, gemm_tc_kernel<1>, tw, tx, p);
    if (e != cudaSuccess) return -6;
    if (p.splits > 1) {
        const size_t total4 = size_t(T) * N / 4;
        int blocks = int((total4 + 255) / 256);
        if (blocks > kNumSMs * 8) blocks = kNumSMs * 8;
        e = launch_pdl(splitk_reduce_kernel, dim3(blocks), dim3(256), 0, stream, (const float*)workspace,
                       p.splits, T, N, epi, out_bf16, resid, out_f32);
        if (e != cudaSuccess) return -6;
    }
    return 0;
}

int gemm_weight_init(GemmWeight* w, const __nv_bfloat16* data, int N, int K) {
    w->data = data;
    w->N = N;
    w->K = K;
    return make_tmap_2d_bf16(w->tmap, data, N, K, kBM, kBK);
}

// Forces the module holding the kernels to load now (lazy loading would otherwise load it at the
// first launch, which can wait on in-flight work such as a spinning NCCL receive).
void preload_gemm() {
    cudaFuncAttributes a;
    cudaFuncGetAttributes(&a, gemm_tc_kernel<1>);
    cudaFuncGetAttributes(&a, gemm_tc_kernel<2>);
    cudaFuncGetAttributes(&a, splitk_reduce_kernel);
    cudaFuncSetAttribute(gemm_tc_kernel<1>, cudaFuncAttributeMaxDynamicSharedMemorySize, kSmemBudget + 2048);
    cudaFuncSetAttribute(gemm_tc_kernel<2>, cudaFuncAttributeMaxDynamicSharedMemorySize, kSmemBudget + 2048);
}

}  // namespace ds
