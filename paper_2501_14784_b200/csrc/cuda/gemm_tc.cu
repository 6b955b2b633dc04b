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
// * Data-parallel + stream-K: whole waves of cluster tiles go to clusters round-robin; the
//   remaining tiles' (tile x k-block) iterations are cut into equal contiguous ranges, one per
//   cluster (no wave quantisation). A tile split across clusters parks fp32 partials; after
//   their main loops its contributors wait for the tile's counter, then each reduces its share
//   of the tile's columns (partials summed in cluster order: deterministic) and applies the
//   epilogue. No separate reduction kernel.
// * TMEM holds two accumulators when the token block fits 256 columns, so a tile's epilogue
//   overlaps the next tile's MMAs.
// * Epilogue: tcgen05.ld -> shared-memory transpose -> 16-byte coalesced stores, fused
//   bf16 / residual-add (x = bf16(x + bf16(acc))) / fp32 (logits).
// * Programmatic dependent launch: the first weight tiles are fetched before waiting on the
//   previous kernel; the activations after.
//
// Warp roles (256 threads): w0 TMA producer, w1 MMA issuer, w2 TMEM allocator, w4..w7 epilogue.
#include <cuda.h>

#include <cstdlib>

#include "common.cuh"
#include "kernels.h"

namespace ds {

constexpr int kBM = 128;      // weight rows per CTA tile (UMMA M)
constexpr int kBK = 64;       // K elements per stage = one 128-byte swizzle row
constexpr int kMaxTB = 512;   // tokens per block (TMEM columns)
constexpr int kCN = 2;        // CTAs per cluster
constexpr int kGemmThreads = 256;
constexpr int kSmemBudget = 200 * 1024;
constexpr int kStageStride = 36;  // floats per row of the epilogue transpose buffer
constexpr int kMaxCounters = 16384;

struct GemmParams {
    int T, N, K;
    int m_tiles;  // N / 128
    int t_blocks;
    int tb;       // tokens per block (<= 512)
    int tb_pad;   // tb rounded up to 16
    int brows;    // activation rows each CTA of the cluster loads per stage (tb_pad / 2)
    int stages;
    int n_acc;    // TMEM accumulators
    int KB;       // k-blocks per tile
    int n_clusters;
    long long dp_tiles;  // cluster tiles handled whole, round-robin
    long long sk_total;  // stream-K iterations (tiles after dp_tiles, x KB)
    int epi;
    __nv_bfloat16* out_bf16;
    const __nv_bfloat16* resid;
    float* out_f32;
    float* partial;  // [n_clusters * 2 CTAs][2 slots][tb_pad/4][128 lanes][4]
    int* counters;   // per CTA tile, zero between launches
};

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
DS_DEVICE void named_bar(int id, int n) { asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(n) : "memory"); }

__host__ __device__ inline long long range_start(long long total, int n, int c) {
    return total * c / n;
}
DS_DEVICE int cluster_of(long long total, int n, long long x) {
    int c = int((x * n) / total);
    while (c + 1 < n && range_start(total, n, c + 1) <= x) ++c;
    while (c > 0 && range_start(total, n, c) > x) --c;
    return c;
}

// A cluster's work in order: its data-parallel tiles, then its stream-K range.
struct Seg {
    long long ut;
    int kb0, kb1;
    bool sk;
};
struct SegIter {
    long long dp_next, dp_end, it, end, sk_base;
    int nc, KB;
    DS_DEVICE SegIter(const GemmParams& p, int c) {
        nc = p.n_clusters;
        KB = p.KB;
        dp_next = c;
        dp_end = p.dp_tiles;
        sk_base = p.dp_tiles * p.KB;
        it = sk_base + range_start(p.sk_total, nc, c);
        end = sk_base + range_start(p.sk_total, nc, c + 1);
    }
    DS_DEVICE bool next(Seg& s) {
        if (dp_next < dp_end) {
            s = {dp_next, 0, KB, false};
            dp_next += nc;
            return true;
        }
        if (it < end) {
            s.ut = it / KB;
            s.kb0 = int(it - s.ut * KB);
            s.kb1 = int(end - it < (long long)(KB - s.kb0) ? s.kb0 + (end - it) : KB);
            s.sk = true;
            it += s.kb1 - s.kb0;
            return true;
        }
        return false;
    }
};

// Applies the epilogue to 16 consecutive token columns of one 32-feature slice held as vals[16]
// (this thread's feature, columns c0..c0+15), through a per-warp transpose buffer.
DS_DEVICE void epilogue16(const GemmParams& p, float* stage, const float* vals, int lane, int t0,
                          int c0, int t_here, int f_base) {
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
        if (p.epi == EPI_F32) {
            float4* dst = reinterpret_cast<float4*>(p.out_f32 + o);
#pragma unroll
            for (int i = 0; i < 4; ++i) dst[i] = make_float4(v[4 * i], v[4 * i + 1], v[4 * i + 2], v[4 * i + 3]);
        } else {
            if (p.epi == EPI_RESID) {
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
    int* last_flag = reinterpret_cast<int*>(tmem_slot + 1);

    const int warp = threadIdx.x >> 5;
    const int lane = threadIdx.x & 31;
    const uint32_t rank = cluster_rank();
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
    cluster_sync();  // remote barriers initialised before any multicast lands
    tc_fence_after();
    const uint32_t tmem_base = *tmem_slot;
    pdl_launch_dependents();

    const int cl_tiles = p.m_tiles / CN;

    if (warp == 0) {
        if (elect_one()) {
            const uint64_t pol_w = policy_evict_first();
            const uint16_t mask = (1u << CN) - 1;
            // weights first (independent of the previous kernel), activations after pdl_wait
            int pre = 0;
            {
                SegIter si(p, cluster);
                Seg sg;
                while (pre < p.stages && si.next(sg)) {
                    const int mt = int(sg.ut % cl_tiles) * CN + int(rank);
                    for (int kb = sg.kb0; kb < sg.kb1 && pre < p.stages; ++kb, ++pre) {
                        mbar_arrive_expect_tx(&full_bar[pre], stage_bytes);
                        tma_load_2d_hint(smem + pre * stage_bytes, &tmap_w, &full_bar[pre], kb * kBK,
                                         mt * kBM, pol_w);
                    }
                }
            }
            pdl_wait();
            int i = 0;
            SegIter si(p, cluster);
            Seg sg;
            while (si.next(sg)) {
                const int tbk = int(sg.ut / cl_tiles);
                const int mt = int(sg.ut % cl_tiles) * CN + int(rank);
                for (int kb = sg.kb0; kb < sg.kb1; ++kb, ++i) {
                    const int s = i % p.stages;
                    const uint32_t round = i / p.stages;
                    uint8_t* sa = smem + s * stage_bytes;
                    uint8_t* sb = sa + a_bytes;
                    if (i >= pre) {
                        mbar_wait(&empty_bar[s], (round & 1) ^ 1);
                        mbar_arrive_expect_tx(&full_bar[s], stage_bytes);
                        tma_load_2d_hint(sa, &tmap_w, &full_bar[s], kb * kBK, mt * kBM, pol_w);
                    }
                    tma_load_2d_mc(sb + rank * p.brows * kBK * 2, &tmap_x, &full_bar[s], kb * kBK,
                                   tbk * p.tb + int(rank) * p.brows, mask);
                }
            }
            // drain: every stage released by both CTAs (no remote arrival after we exit)
            const int n = i;
            for (int k = (n > p.stages ? n - p.stages : 0); k < n; ++k)
                mbar_wait(&empty_bar[k % p.stages], (uint32_t(k / p.stages) & 1));
        }
    } else if (warp == 1) {
        int i = 0, seg = 0;
        SegIter si(p, cluster);
        Seg sg;
        while (si.next(sg)) {
            const int tbk = int(sg.ut / cl_tiles);
            const int t_here = min(p.tb, p.T - tbk * p.tb);
            const int a = seg % p.n_acc;
            const uint32_t acc = tmem_base + uint32_t(a * 256);
            mbar_wait(&tempty_bar[a], ((seg / p.n_acc) & 1) ^ 1);
            tc_fence_after();
            for (int kb = sg.kb0; kb < sg.kb1; ++kb, ++i) {
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
                                      (kb > sg.kb0 || k > 0) ? 1u : 0u);
                    }
                    umma_commit_mc(&empty_bar[s], (1u << CN) - 1);
                    if (kb == sg.kb1 - 1) umma_commit(&tfull_bar[a]);
                }
                __syncwarp();
            }
            ++seg;
        }
    } else if (warp >= 4) {
        pdl_wait();
        const int q = warp & 3;
        const int tid = threadIdx.x - 128;  // 0..127, = TMEM lane
        float* stage = ep_stage + q * 16 * kStageStride;
        const size_t slot_floats = size_t(p.tb_pad) * kBM;
        int seg = 0;
        bool first_sk = true;
        long long pending[2];  // split tiles this CTA parked a partial for (<= 2 per range)
        int n_pending = 0;
        SegIter si(p, cluster);
        Seg sg;
        while (si.next(sg)) {
            const int tbk = int(sg.ut / cl_tiles);
            const int mt = int(sg.ut % cl_tiles) * CN + int(rank);
            const int t0 = tbk * p.tb;
            const int t_here = min(p.tb, p.T - t0);
            const int a = seg % p.n_acc;
            const uint32_t acc = tmem_base + uint32_t(a * 256) + (uint32_t(q * 32) << 16);
            mbar_wait(&tfull_bar[a], (seg / p.n_acc) & 1);
            tc_fence_after();
            if (sg.kb0 == 0 && sg.kb1 == p.KB) {
                for (int c0 = 0; c0 < t_here; c0 += 16) {
                    uint32_t r[16];
                    tmem_ld16(acc + c0, r);
                    tmem_ld_wait();
                    epilogue16(p, stage, reinterpret_cast<float*>(r), lane, t0, c0, t_here,
                               mt * kBM + q * 32);
                }
                tc_fence_before();
                __syncwarp();
                if (lane == 0) mbar_arrive(&tempty_bar[a]);
            } else {
                // park the partial as [col/4][lane][4] (16-byte stores, 512 B per warp)
                const int slot = first_sk ? 0 : 1;
                float4* mine = reinterpret_cast<float4*>(
                    p.partial + (size_t(cluster * CN + rank) * 2 + slot) * slot_floats);
                for (int c0 = 0; c0 < t_here; c0 += 16) {
                    uint32_t r[16];
                    tmem_ld16(acc + c0, r);
                    tmem_ld_wait();
#pragma unroll
                    for (int jj = 0; jj < 4; ++jj)
                        mine[size_t(c0 / 4 + jj) * kBM + tid] =
                            make_float4(__uint_as_float(r[4 * jj]), __uint_as_float(r[4 * jj + 1]),
                                        __uint_as_float(r[4 * jj + 2]), __uint_as_float(r[4 * jj + 3]));
                }
                tc_fence_before();
                __syncwarp();
                if (lane == 0) mbar_arrive(&tempty_bar[a]);  // accumulator free for the next tile
                __threadfence();
                named_bar(1, 128);
                if (tid == 0) atomicAdd(&p.counters[int(sg.ut) * CN + int(rank)], 1);
                pending[n_pending++] = sg.ut;  // reduced after the main loop, in parallel
            }
            if (sg.sk) first_sk = false;
            ++seg;
        }
        // Deferred, parallel fixup: every contributor of a split tile waits until all partials
        // are parked, then reduces its share of the tile's 16-column chunks (partials summed in
        // cluster order: deterministic) and applies the epilogue. Waiting only at the end keeps
        // the stream-K ranges from serialising on each other.
        for (int pi = 0; pi < n_pending; ++pi) {
            const long long ut = pending[pi];
            const int tbk = int(ut / cl_tiles);
            const int mt = int(ut % cl_tiles) * CN + int(rank);
            const int t0 = tbk * p.tb;
            const int t_here = min(p.tb, p.T - t0);
            const long long x_lo = ut * p.KB - p.dp_tiles * p.KB;
            const long long x_hi = x_lo + p.KB - 1;
            const int c_lo = cluster_of(p.sk_total, p.n_clusters, x_lo);
            const int c_hi = cluster_of(p.sk_total, p.n_clusters, x_hi);
            const int nseg = c_hi - c_lo + 1;
            const int ctr = int(ut) * CN + int(rank);
            if (tid == 0) {
                volatile int* cnt = p.counters + ctr;
                while (*cnt < nseg) __nanosleep(100);
            }
            named_bar(1, 128);
            __threadfence();
            const int nch = (t_here + 15) / 16;
            const int k = cluster - c_lo;
            const int ch0 = k * nch / nseg, ch1 = (k + 1) * nch / nseg;
            {
                {
                    for (int c0 = ch0 * 16; c0 < ch1 * 16; c0 += 16) {
                        float v[16];
#pragma unroll
                        for (int j = 0; j < 16; ++j) v[j] = 0.f;
                        for (int cb = c_lo; cb <= c_hi; cb += 4) {
                            float4 buf[4][4];
#pragma unroll
                            for (int u = 0; u < 4; ++u) {
                                const int c = cb + u;
                                if (c > c_hi) break;
                                const int sl = range_start(p.sk_total, p.n_clusters, c) >= x_lo ? 0 : 1;
                                const float4* src = reinterpret_cast<const float4*>(
                                    p.partial + (size_t(c * CN + rank) * 2 + sl) * slot_floats);
#pragma unroll
                                for (int jj = 0; jj < 4; ++jj)
                                    buf[u][jj] = __ldcg(src + size_t(c0 / 4 + jj) * kBM + tid);
                            }
#pragma unroll
                            for (int u = 0; u < 4; ++u) {
                                if (cb + u > c_hi) break;
#pragma unroll
                                for (int jj = 0; jj < 4; ++jj) {
                                    v[4 * jj] += buf[u][jj].x;
                                    v[4 * jj + 1] += buf[u][jj].y;
                                    v[4 * jj + 2] += buf[u][jj].z;
                                    v[4 * jj + 3] += buf[u][jj].w;
                                }
                            }
                        }
                        epilogue16(p, stage, v, lane, t0, c0, t_here, mt * kBM + q * 32);
                    }
                }
            }
            // the last contributor to finish resets both counters for the next launch
            named_bar(1, 128);
            if (tid == 0) {
                int* done = p.counters + kMaxCounters;
                if (atomicAdd(done + ctr, 1) == nseg - 1) {
                    p.counters[ctr] = 0;
                    done[ctr] = 0;
                }
            }
        }
    }
    __syncthreads();
    cluster_sync();
    if (warp == 2) {
        tc_fence_after();
        tmem_dealloc(tmem_base, 512);
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

// partials for every CTA (2 slots of 128 x 512 fp32) + per-tile counters (zero-initialised)
size_t gemm_workspace_floats() { return size_t(kNumSMs) * 2 * kBM * kMaxTB + 2 * kMaxCounters; }

int gemm_bf16(const GemmWeight& w, const __nv_bfloat16* x, int T, int epi, __nv_bfloat16* out_bf16,
              const __nv_bfloat16* resid, float* out_f32, float* workspace, size_t workspace_floats,
              int max_clusters, cudaStream_t stream) {
    const int N = w.N, K = w.K;
    if (T <= 0) return 0;
    static const int cn_env = getenv("DS_GEMM_CN") ? atoi(getenv("DS_GEMM_CN")) : kCN;
    const int cn = (cn_env == 1 || (N / kBM) % 2 != 0) ? 1 : 2;
    if (K % kBK != 0 || N % kBM != 0) return -3;
    if (!workspace || workspace_floats < gemm_workspace_floats()) return -7;
    GemmParams p{};
    p.T = T;
    p.N = N;
    p.K = K;
    p.m_tiles = N / kBM;
    p.t_blocks = (T + kMaxTB - 1) / kMaxTB;
    if (p.t_blocks * p.m_tiles > kMaxCounters) return -8;
    p.tb = T < kMaxTB ? T : kMaxTB;
    p.tb_pad = (p.tb + 15) & ~15;
    p.brows = p.tb_pad / cn;
    p.KB = K / kBK;
    const int stage_bytes = kBM * kBK * 2 + p.tb_pad * kBK * 2;
    const int fixed = 4 * 16 * kStageStride * 4 + 256 + 1024;
    p.stages = (kSmemBudget - fixed) / stage_bytes;
    if (p.stages > 8) p.stages = 8;
    if (p.stages < 2) return -4;
    p.n_acc = p.tb_pad <= 256 ? 2 : 1;
    const long long tiles = (long long)p.t_blocks * (p.m_tiles / cn);
    int nc = kNumSMs / cn;
    if (max_clusters > 0 && nc > max_clusters) nc = max_clusters;
    // whole waves data-parallel; the remainder stream-K with >= 8 k-blocks per cluster
    long long dp = tiles >= nc ? (tiles / nc) * nc : 0;
    if (dp == tiles) {
        // exact waves: nothing to split
    } else if ((tiles - dp) * p.KB < 8LL * nc && dp >= nc) {
        dp -= nc;  // tiny remainder: fold the last full wave into the stream-K part
    }
    long long sk = (tiles - dp) * p.KB;
    if (dp == 0 && sk > 0 && sk / 4 < nc) nc = int(sk / 4 > 0 ? sk / 4 : 1);  // tiny GEMM: fewer clusters
    if (dp > 0 && nc > tiles) nc = int(tiles);
    p.n_clusters = nc;
    p.dp_tiles = dp;
    p.sk_total = sk;
    p.epi = epi;
    p.out_bf16 = out_bf16;
    p.resid = resid;
    p.out_f32 = out_f32;
    p.partial = workspace;
    p.counters = reinterpret_cast<int*>(workspace + size_t(kNumSMs) * 2 * kBM * kMaxTB);
    alignas(64) CUtensorMap tx;
    if (make_tmap_2d_bf16(&tx, x, T, K, p.brows, kBK) != 0) return -5;
    const size_t smem = size_t(p.stages) * stage_bytes + fixed;
    cudaLaunchConfig_t cfg{};
    cfg.gridDim = dim3(nc * cn);
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
    cudaError_t e = cn == 2 ? cudaLaunchKernelEx(&cfg, gemm_tc_kernel<2>,
                                                 *reinterpret_cast<const CUtensorMap*>(w.tmap), tx, p)
                            : cudaLaunchKernelEx(&cfg, gemm_tc_kernel<1>,
                                                 *reinterpret_cast<const CUtensorMap*>(w.tmap), tx, p);
    return e == cudaSuccess ? 0 : -6;
}

int gemm_weight_init(GemmWeight* w, const __nv_bfloat16* data, int N, int K) {
    w->data = data;
    w->N = N;
    w->K = K;
    return make_tmap_2d_bf16(w->tmap, data, N, K, kBM, kBK);
}

// Forces the module holding the kernel to load now (lazy loading would otherwise load it at the
// first launch, which can wait on in-flight work such as a spinning NCCL receive).
void preload_gemm() {
    cudaFuncAttributes a;
    cudaFuncGetAttributes(&a, gemm_tc_kernel<1>);
    cudaFuncGetAttributes(&a, gemm_tc_kernel<2>);
    cudaFuncSetAttribute(gemm_tc_kernel<1>, cudaFuncAttributeMaxDynamicSharedMemorySize, kSmemBudget + 2048);
    cudaFuncSetAttribute(gemm_tc_kernel<2>, cudaFuncAttributeMaxDynamicSharedMemorySize, kSmemBudget + 2048);
}

}  // namespace ds
