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
// * Persistent clusters, hybrid data-parallel + stream-K schedule: whole waves of cluster tiles
//   are dealt one per cluster; the remaining (tile, k-block) iteration space is cut into equal
//   contiguous ranges, one per cluster, so every SM streams the same number of weight bytes.
//   A tile split across clusters is finished by its LAST-arriving CTA (per-tile arrival counter):
//   the others park fp32 pieces in a workspace slot and move on; nobody waits, and the finisher
//   sums the pieces in k order (deterministic) into the fused epilogue. (A designated-owner fixup
//   and a separate split-K reduction kernel were both measured slower.)
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
constexpr int kSkPieces = 8;  // stream-K pieces per remainder tile (0: uncapped); DS_GEMM_SKP
constexpr int kGemmThreads = 256;
constexpr int kSmemBudget = 222 * 1024;
constexpr int kStageStride = 36;  // floats per row of the epilogue transpose buffer
constexpr size_t kWorkspaceFloats = size_t(24) << 20;  // arrival counters + stream-K pieces
constexpr size_t kCounterInts = size_t(64) << 10;
constexpr int kRsMax = 1024;  // token rows a consumer GEMM can scale (RowNorm)
constexpr int kRsFloats = 4 * kMaxTB;  // RowNorm smem: consumer scales [kRsMax] / producer slices [4][kMaxTB]
constexpr int kFixedSmem = 4 * 16 * kStageStride * 4 + 256 + kRsFloats * 4 + 1024;  // transpose buffers,
                                                                                  // barriers, RowNorm, align

struct GemmParams {
    int T, N, K;
    int m_tiles;  // N / 128
    int t_blocks;
    int tb;       // tokens per block (<= 512)
    int tb_pad;   // tb rounded up to 16
    int brows;    // activation rows per TMA box (tb_pad / CN; 2-SM: half an instruction's N)
    int b_bytes;  // activation bytes per stage in each CTA's shared memory
    int two_sm;   // 1: CTA pair runs tcgen05.mma.cta_group::2 (M = 256, B split by columns)
    int tb_fast;  // 1: tile index runs token blocks fastest (token-split narrow GEMMs: the blocks
                  //    sharing a weight tile stream it concurrently, L2 serves the re-reads)
    int stages;
    int n_acc;    // TMEM accumulators
    int KB;       // k-blocks per tile
    int n_clusters;
    int dp_rounds;  // whole-tile rounds (tile = round * n_clusters + cluster)
    int sk_tiles;   // tiles after the data-parallel rounds, shared out by k-block ranges
    int n_sk;       // clusters taking a stream-K range (<= sk_tiles * KB: no empty range)
    int defer;      // 1: split tiles are summed by splitk_finish_kernel instead of the last arriver
    int planes;     // > 0: aligned narrow GEMM, partials in [planes][T][N] for splitk_reduce_kernel
    int ks;         // > 1: narrow GEMM, K split ks ways INSIDE each cluster (CN x ks CTAs, one
                    // tile per cluster), partials summed through distributed shared memory
    int epi;
    __nv_bfloat16* out_bf16;
    const __nv_bfloat16* resid;
    float* out_f32;
    float* slots;   // [n_clusters][2][CN][tb_pad][128] fp32 pieces of split tiles
    int* counters;  // [tiles][CN] arrivals (self-resetting)
    unsigned long long* trace;  // optional per-CTA phase timestamps (gemm_set_trace)
    const __nv_bfloat16* w;     // weight base (L2 prefetch addresses)
    int pf_kb;                  // k-blocks per CTA to prefetch into L2 past the smem pipeline
    int ks_push;                // k-split epilogue: peers push row blocks with bulk DSMEM copies
    // RMSNorm split across the residual GEMM and its consumer (RowNorm):
    float* ssq_out;       // producer (EPI_RESID): sums of squares of its output row slices
                          // [m_tiles][T] (one per 128-feature tile)
    const float* rs_ssq;  // consumer: those parts; out row t is scaled by
    int rs_parts;         //   r[t] = 1 / sqrt(sum of its rs_parts parts / rs_d + rs_eps)
    int rs_d;
    float rs_eps;
    float* rs_out;        // consumer with deferred planes: CTA 0 publishes the row scales [T]
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

DS_DEVICE void prefetch_l2_bulk(const void* p, uint32_t bytes) {
    asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(reinterpret_cast<uint64_t>(p)), "r"(bytes)
                 : "memory");
}

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

// A segment: cluster tile ut, k-blocks [kb0, kb1), and (stream-K part) which of this cluster's two
// piece slots it would use.
struct Seg {
    int ut, kb0, kb1, which;
};
// Token block and (cluster-level) feature tile of tile index ut.
DS_DEVICE int tile_tbk(const GemmParams& p, int ut, int cl_tiles) {
    return p.tb_fast ? ut % p.t_blocks : ut / cl_tiles;
}
DS_DEVICE int tile_mtc(const GemmParams& p, int ut, int cl_tiles) {
    return p.tb_fast ? ut / p.t_blocks : ut % cl_tiles;
}

// Stream-K range of cluster c over the sk_tiles * KB iteration space.
DS_DEVICE int sk_begin(const GemmParams& p, int c) {
    return int((long long)c * p.sk_tiles * p.KB / p.n_sk);
}
// Cluster whose stream-K range holds iteration g.
DS_DEVICE int sk_owner(const GemmParams& p, int g) {
    const long long G = (long long)p.sk_tiles * p.KB;
    return int(((long long)(g + 1) * p.n_sk + G - 1) / G) - 1;
}
// Iterates this cluster's segments: its stream-K range over tiles [0, sk_tiles) first (so split
// tiles are finished while the data-parallel tiles stream), then one tile per data-parallel round.
template <typename F>
DS_DEVICE void for_each_seg(const GemmParams& p, int cluster, int kidx, F&& f) {
    if (p.ks > 1) {  // k-split cluster: tile `cluster`, this CTA's share of its k-blocks
        f(Seg{cluster, kidx * p.KB / p.ks, (kidx + 1) * p.KB / p.ks, 0});
        return;
    }
    if (cluster < p.n_sk) {
        const int g0 = sk_begin(p, cluster), g1 = sk_begin(p, cluster + 1);
        for (int g = g0; g < g1;) {
            const int t = g / p.KB, kb0 = g % p.KB;
            const int kb1 = min(p.KB, kb0 + (g1 - g));
            f(Seg{t, kb0, kb1, g == g0 ? 0 : 1});
            g += kb1 - kb0;
        }
    }
    for (int r = 0; r < p.dp_rounds; ++r) f(Seg{p.sk_tiles + r * p.n_clusters + cluster, 0, p.KB, 0});
}

// Transposes 16 consecutive token columns of one 32-feature slice (vals[16]: this thread's
// feature, columns c0..c0+15) through a per-warp buffer: afterwards the thread holds token row
// lane/2, features (lane&1)*16 .. +15 of the slice in v[16]. Returns false for padding rows.
DS_DEVICE bool transpose16(float* stage, const float* vals, int lane, int c0, int t_here, float* v) {
#pragma unroll
    for (int j = 0; j < 16; ++j) stage[j * kStageStride + lane] = vals[j];
    __syncwarp();
    const int row = lane >> 1, half = lane & 1;
    const bool ok = c0 + row < t_here;
    if (ok) {
        const float4* src = reinterpret_cast<const float4*>(stage + row * kStageStride + half * 16);
#pragma unroll
        for (int i = 0; i < 4; ++i) {
            const float4 x = src[i];
            v[4 * i] = x.x;
            v[4 * i + 1] = x.y;
            v[4 * i + 2] = x.z;
            v[4 * i + 3] = x.w;
        }
    }
    __syncwarp();
    return ok;
}

// Final epilogue of 16 features f0.. of token row t: bf16 / residual-add / fp32 store.
DS_DEVICE void store16(const GemmParams& p, float* v, int t, int f0) {
    const size_t o = size_t(t) * p.N + f0;
    if (p.epi == EPI_F32) {
        float4* dst = reinterpret_cast<float4*>(p.out_f32 + o);
#pragma unroll
        for (int i = 0; i < 4; ++i) dst[i] = make_float4(v[4 * i], v[4 * i + 1], v[4 * i + 2], v[4 * i + 3]);
        return;
    }
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

// SiLU epilogue of one transposed 32-feature slice f_slice.. (16 gate + the matching 16 up rows
// of the interleaved weight): lane 2r holds the gate, lane 2r+1 the up features of token row r;
// they swap halves and each writes 8 of the 16 ffn columns. Every lane must call (shuffles).
DS_DEVICE void store_silu(const GemmParams& p, const float* v, bool ok, int lane, int t, int f_slice) {
    const int half = lane & 1;
    float send[8], recv[8];
#pragma unroll
    for (int j = 0; j < 8; ++j) send[j] = half ? v[j] : v[8 + j];
#pragma unroll
    for (int j = 0; j < 8; ++j) recv[j] = __shfl_xor_sync(0xffffffffu, send[j], 1);
    if (!ok) return;
    const float* g = half ? recv : v;
    const float* u = half ? v + 8 : recv;
    float o[8];
#pragma unroll
    for (int j = 0; j < 8; ++j) {
        const float gb = round_bf(g[j]);
        o[j] = round_bf(__fdividef(gb, 1.0f + __expf(-gb))) * round_bf(u[j]);  // fast math: bf16-rounded
    }
    const int ld = p.N / 2;
    *reinterpret_cast<uint4*>(p.out_bf16 + size_t(t) * ld + (f_slice / 32) * 16 + half * 8) = pack8(o);
}

// Final epilogue of a transposed chunk (all lanes call; `ok` = this lane's token row is real);
// sc = the row's RMSNorm scale (RowNorm consumer) or 1.
DS_DEVICE void epi_store(const GemmParams& p, float* v, bool ok, int lane, int t, int f_slice, float sc = 1.f) {
    if (p.rs_ssq) {
#pragma unroll
        for (int j = 0; j < 16; ++j) v[j] *= sc;
    }
    if (p.epi == EPI_SILU) {
        store_silu(p, v, ok, lane, t, f_slice);
        return;
    }
    if (ok) store16(p, v, t, f_slice + (lane & 1) * 16);
}

DS_DEVICE void epi_bar() { asm volatile("bar.sync 1, 128;" ::: "memory"); }

// Piece slot of cluster c for the split tile starting at k-block tile_g0 (its first or last
// stream-K segment), plus this thread's offset.
DS_DEVICE const float* piece_ptr(const GemmParams& p, int cn, int rank, int c, int tile_g0, size_t off) {
    const int which = sk_begin(p, c) >= tile_g0 ? 0 : 1;
    return p.slots + ((size_t(c) * 2 + which) * cn + rank) * (size_t(p.tb_pad) * kBM) + off;
}

// sum[16] = the 16 values at `off` of every piece of a split tile, added in cluster (= k) order;
// the finishing cluster `self` contributes `own` (its TMEM values) at its position; kPieceBatch
// pieces' loads are in flight at a time.
constexpr int kPieceBatch = 2;
DS_DEVICE void sum_pieces(const GemmParams& p, int cn, int rank, int tile_g0, int c_lo, int c_hi,
                          size_t off, int self, const float* own, float* sum) {
#pragma unroll
    for (int j = 0; j < 16; ++j) sum[j] = 0.f;
    for (int cb = c_lo; cb <= c_hi; cb += kPieceBatch) {
        float4 x[kPieceBatch][4];
#pragma unroll
        for (int i = 0; i < kPieceBatch; ++i) {
            const int c = cb + i;
            if (c <= c_hi && c != self) {
                const float4* src = reinterpret_cast<const float4*>(piece_ptr(p, cn, rank, c, tile_g0, off));
#pragma unroll
                for (int k = 0; k < 4; ++k) x[i][k] = __ldcg(src + k);
            }
        }
#pragma unroll
        for (int i = 0; i < kPieceBatch; ++i) {
            const int c = cb + i;
            if (c > c_hi) break;
            if (c == self) {
#pragma unroll
                for (int j = 0; j < 16; ++j) sum[j] += own[j];
            } else {
#pragma unroll
                for (int k = 0; k < 4; ++k) {
                    sum[4 * k] += x[i][k].x;
                    sum[4 * k + 1] += x[i][k].y;
                    sum[4 * k + 2] += x[i][k].z;
                    sum[4 * k + 3] += x[i][k].w;
                }
            }
        }
    }
}

DS_DEVICE uint32_t mapa_shared(uint32_t addr, uint32_t cta) {
    uint32_t r;
    asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(r) : "r"(addr), "r"(cta));
    return r;
}
DS_DEVICE float4 ld_dsmem_f4(uint32_t addr) {
    float4 v;
    asm volatile("ld.shared::cluster.v4.f32 {%0,%1,%2,%3}, [%4];"
                 : "=f"(v.x), "=f"(v.y), "=f"(v.z), "=f"(v.w)
                 : "r"(addr)
                 : "memory");
    return v;
}
DS_DEVICE void add4(float4& a, const float4& b) {
    a.x += b.x;
    a.y += b.y;
    a.z += b.z;
    a.w += b.w;
}

DS_DEVICE void bulk_s2cluster(uint32_t dst_cluster, uint32_t src, uint32_t bytes, uint32_t bar_cluster) {
    asm volatile(
        "cp.async.bulk.shared::cluster.shared::cta.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
            dst_cluster),
        "r"(src), "r"(bytes), "r"(bar_cluster)
        : "memory");
}
DS_DEVICE void bulk_commit() { asm volatile("cp.async.bulk.commit_group;" ::: "memory"); }
DS_DEVICE void bulk_wait_read0() { asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory"); }
DS_DEVICE void fence_async_smem() { asm volatile("fence.proxy.async.shared::cta;" ::: "memory"); }

constexpr int kPushWin = 128;  // token rows per window of the push epilogue

// Shared memory the push epilogue needs: the parked window + (ks - 1) received row blocks + a barrier.
inline size_t ksplit_push_smem(int ks) {
    const size_t rows = size_t((kPushWin + ks - 1) / ks);
    return size_t(kPushWin) * kBM * 4 + size_t(ks - 1) * rows * kBM * 4 + 64;
}

// k-split cluster epilogue, push form: every CTA parks a window of <= 128 token columns, then
// ONE thread sends each peer its row block with a bulk shared::cta -> shared::cluster copy (the
// copy engine moves it; completion on the peer's mbarrier), and each CTA sums its own rows from
// local shared memory in k order (deterministic, as the pull form) and applies the epilogue.
template <int CN>
DS_DEVICE void ksplit_epilogue_push(const GemmParams& p, uint8_t* smem, uint32_t tmem_base, int cluster,
                                    int kidx, int rank, int warp, int lane) {
    const int cl_tiles = p.m_tiles / CN;
    const int tbk = tile_tbk(p, cluster, cl_tiles);
    const int mt = tile_mtc(p, cluster, cl_tiles) * CN + rank;
    const int t0 = tbk * p.tb;
    const int t_here = min(p.tb, p.T - t0);
    const int ks = p.ks;
    const int max_rows = (kPushWin + ks - 1) / ks;
    float* part = reinterpret_cast<float*>(smem);              // [128 tokens][128 features]
    float* recv = part + size_t(kPushWin) * kBM;               // [ks - 1][max_rows][128]
    uint64_t* bar = reinterpret_cast<uint64_t*>(recv + size_t(ks - 1) * max_rows * kBM);
    const int quarter = warp & 3, cgrp = warp >> 2;
    const bool silu = p.epi == EPI_SILU;
    const int ipr = silu ? 16 : 32;
    if (threadIdx.x == 0) {
        mbar_init(bar, 1);
        fence_mbar_init();
    }
    int phase = 0;
    for (int w0 = 0; w0 < t_here; w0 += kPushWin, phase ^= 1) {
        const int wn = min(kPushWin, t_here - w0);
        for (int c = cgrp * 16; c < wn; c += 32) {
            uint32_t r[16];
            tmem_ld16(tmem_base + (uint32_t(quarter * 32) << 16) + uint32_t(w0 + c), r);
            tmem_ld_wait();
#pragma unroll
            for (int j = 0; j < 16; ++j) part[(c + j) * kBM + quarter * 32 + lane] = __uint_as_float(r[j]);
        }
        if (threadIdx.x == 128 && w0 == 0) GEMM_TRACE(6);
        // every CTA parked (and done reading its receive buffers of the previous window)
        cluster_sync();
        if (threadIdx.x == 128 && w0 == 0) GEMM_TRACE(7);
        const int r0 = kidx * wn / ks, r1 = (kidx + 1) * wn / ks;
        if (threadIdx.x == 0) {
            fence_async_smem();  // the parked window (generic writes) is the copies' source
            mbar_arrive_expect_tx(bar, uint32_t((ks - 1) * (r1 - r0) * kBM * 4));
            for (int k = 0; k < ks; ++k) {
                if (k == kidx) continue;
                const int q0 = k * wn / ks, q1 = (k + 1) * wn / ks;  // peer k's rows
                if (q1 <= q0) continue;
                const int slot = kidx < k ? kidx : kidx - 1;         // my block in peer k's recv
                const uint32_t peer = uint32_t(k * CN + rank);
                const uint32_t dst = mapa_shared(smem_u32(recv + size_t(slot) * max_rows * kBM), peer);
                bulk_s2cluster(dst, smem_u32(part + size_t(q0) * kBM), uint32_t((q1 - q0) * kBM * 4),
                               mapa_shared(smem_u32(bar), peer));
            }
            bulk_commit();
        }
        mbar_wait(bar, uint32_t(phase));  // the peers' blocks of my rows landed
        for (int it = threadIdx.x; it < (r1 - r0) * ipr; it += kGemmThreads) {
            const int row = r0 + it / ipr, q4 = it % ipr;
            const int f = silu ? (q4 >> 2) * 32 + (q4 & 3) * 4 : q4 * 4;
            float4 a = make_float4(0.f, 0.f, 0.f, 0.f), u = a;
            for (int k = 0; k < ks; ++k) {  // k order: deterministic
                const float* src = k == kidx ? part + size_t(row) * kBM
                                             : recv + (size_t(k < kidx ? k : k - 1) * max_rows + (row - r0)) * kBM;
                add4(a, *reinterpret_cast<const float4*>(src + f));
                if (silu) add4(u, *reinterpret_cast<const float4*>(src + f + 16));
            }
            const int t = t0 + w0 + row, fg = mt * kBM + f;
            const float v[4] = {a.x, a.y, a.z, a.w};
            if (p.epi == EPI_F32) {
                *reinterpret_cast<float4*>(p.out_f32 + size_t(t) * p.N + fg) = a;
            } else if (silu) {
                const float uu[4] = {u.x, u.y, u.z, u.w};
                float h[4];
#pragma unroll
                for (int j = 0; j < 4; ++j) {
                    const float gb = round_bf(v[j]);
                    h[j] = round_bf(__fdividef(gb, 1.0f + __expf(-gb))) * round_bf(uu[j]);
                }
                uint2 hv;
                hv.x = pack2(h[0], h[1]);
                hv.y = pack2(h[2], h[3]);
                *reinterpret_cast<uint2*>(p.out_bf16 + size_t(t) * (p.N / 2) + (fg / 32) * 16 + fg % 32) = hv;
            } else {
                float o[4] = {v[0], v[1], v[2], v[3]};
                const size_t oi = size_t(t) * p.N + fg;
                if (p.epi == EPI_RESID) {
                    const uint2 rv = *reinterpret_cast<const uint2*>(p.resid + oi);
                    const __nv_bfloat162* rh = reinterpret_cast<const __nv_bfloat162*>(&rv);
                    const float2 x0 = __bfloat1622float2(rh[0]), x1 = __bfloat1622float2(rh[1]);
                    o[0] = x0.x + round_bf(o[0]);
                    o[1] = x0.y + round_bf(o[1]);
                    o[2] = x1.x + round_bf(o[2]);
                    o[3] = x1.y + round_bf(o[3]);
                }
                uint2 ov;
                ov.x = pack2(o[0], o[1]);
                ov.y = pack2(o[2], o[3]);
                *reinterpret_cast<uint2*>(p.out_bf16 + oi) = ov;
            }
        }
        if (threadIdx.x == 0) bulk_wait_read0();  // my window read out before it is re-parked
        __syncthreads();
    }
    cluster_sync();  // every push into this CTA landed and was consumed before anyone exits
}

// k-split cluster epilogue (all 256 threads): the ks CTAs holding the same 128 features park
// their fp32 accumulators in their (now idle) pipeline shared memory, 256 token columns at a
// time, and each sums its 1/ks share of the token rows over the cluster's CTAs in k order
// (ld.shared::cluster), then applies the fused epilogue 4 features per thread.
template <int CN>
DS_DEVICE void ksplit_epilogue(const GemmParams& p, uint8_t* smem, uint32_t tmem_base, int cluster,
                               int kidx, int rank, int warp, int lane, const float* rs) {
    const int cl_tiles = p.m_tiles / CN;
    const int tbk = tile_tbk(p, cluster, cl_tiles);
    const int mt = tile_mtc(p, cluster, cl_tiles) * CN + rank;
    const int t0 = tbk * p.tb;
    const int t_here = min(p.tb, p.T - t0);
    float* part = reinterpret_cast<float*>(smem);  // [256 tokens][128 features]
    const uint32_t part_u32 = smem_u32(part);
    const int quarter = warp & 3, cgrp = warp >> 2;
    const bool silu = p.epi == EPI_SILU;
    const int ipr = silu ? 16 : 32;  // 4-feature items per token row (SiLU: gate quads only)
    for (int w0 = 0; w0 < t_here; w0 += 256) {
        const int wn = min(256, t_here - w0);
        for (int c = cgrp * 16; c < wn; c += 32) {
            uint32_t r[16];
            tmem_ld16(tmem_base + (uint32_t(quarter * 32) << 16) + uint32_t(w0 + c), r);
            tmem_ld_wait();
#pragma unroll
            for (int j = 0; j < 16; ++j) part[(c + j) * kBM + quarter * 32 + lane] = __uint_as_float(r[j]);
        }
        if (threadIdx.x == 128 && w0 == 0) GEMM_TRACE(6);  // window parked
        cluster_sync();  // every CTA's window parked and visible cluster-wide
        if (threadIdx.x == 128 && w0 == 0) GEMM_TRACE(7);  // cluster arrived
        const int r0 = kidx * wn / p.ks, r1 = (kidx + 1) * wn / p.ks;
        for (int it = threadIdx.x; it < (r1 - r0) * ipr; it += kGemmThreads) {
            const int row = r0 + it / ipr, q4 = it % ipr;
            const int f = silu ? (q4 >> 2) * 32 + (q4 & 3) * 4 : q4 * 4;
            float4 a = make_float4(0.f, 0.f, 0.f, 0.f), u = a;
            const uint32_t off = part_u32 + uint32_t((row * kBM + f) * 4);
            for (int k = 0; k < p.ks; ++k) {  // k order: deterministic
                const uint32_t peer = uint32_t(k * CN + rank);
                add4(a, ld_dsmem_f4(mapa_shared(off, peer)));
                if (silu) add4(u, ld_dsmem_f4(mapa_shared(off + 64, peer)));
            }
            const int t = t0 + w0 + row, fg = mt * kBM + f;
            if (p.rs_ssq) {
                const float sc = rs[t];
                a.x *= sc, a.y *= sc, a.z *= sc, a.w *= sc;
                u.x *= sc, u.y *= sc, u.z *= sc, u.w *= sc;
            }
            const float v[4] = {a.x, a.y, a.z, a.w};
            if (p.epi == EPI_F32) {
                *reinterpret_cast<float4*>(p.out_f32 + size_t(t) * p.N + fg) = a;
            } else if (silu) {
                const float uu[4] = {u.x, u.y, u.z, u.w};
                float h[4];
#pragma unroll
                for (int j = 0; j < 4; ++j) {
                    const float gb = round_bf(v[j]);
                    h[j] = round_bf(__fdividef(gb, 1.0f + __expf(-gb))) * round_bf(uu[j]);
                }
                uint2 hv;
                hv.x = pack2(h[0], h[1]);
                hv.y = pack2(h[2], h[3]);
                *reinterpret_cast<uint2*>(p.out_bf16 + size_t(t) * (p.N / 2) + (fg / 32) * 16 + fg % 32) = hv;
            } else {
                float o[4] = {v[0], v[1], v[2], v[3]};
                const size_t oi = size_t(t) * p.N + fg;
                if (p.epi == EPI_RESID) {
                    const uint2 rv = *reinterpret_cast<const uint2*>(p.resid + oi);
                    const __nv_bfloat162* rh = reinterpret_cast<const __nv_bfloat162*>(&rv);
                    const float2 x0 = __bfloat1622float2(rh[0]), x1 = __bfloat1622float2(rh[1]);
                    o[0] = x0.x + round_bf(o[0]);
                    o[1] = x0.y + round_bf(o[1]);
                    o[2] = x1.x + round_bf(o[2]);
                    o[3] = x1.y + round_bf(o[3]);
                }
                uint2 ov;
                ov.x = pack2(o[0], o[1]);
                ov.y = pack2(o[2], o[3]);
                *reinterpret_cast<uint2*>(p.out_bf16 + oi) = ov;
                if (p.ssq_out) {  // one warp = one token row's 128 features of this tile
                    float ss = 0.f;
#pragma unroll
                    for (int j = 0; j < 4; ++j) {
                        const float xb = round_bf(o[j]);  // the stored bf16 of x
                        ss += xb * xb;
                    }
                    ss = warp_sum(ss);
                    if (lane == 0) p.ssq_out[size_t(mt) * p.T + t] = ss;
                }
            }
        }
        cluster_sync();  // peers done reading before the next window overwrites it
    }
}

DS_DEVICE void mbar_arrive_remote(uint32_t cluster_addr) {
    asm volatile("mbarrier.arrive.release.cluster.shared::cluster.b64 _, [%0];" ::"r"(cluster_addr)
                 : "memory");
}

// TWO (CN == 2): the pair runs 2-SM MMAs issued by the even CTA; each CTA stages its own 128
// weight rows and HALF of each instruction's token columns, so a stage costs 16 KB + T/2 rows
// instead of 16 KB + T rows: about twice the pipeline depth at T >= 256.
template <int CN, bool TWO>
__global__ void __maxnreg__(168)  // leaves registers for the co-resident finish kernel
gemm_tc_kernel(const __grid_constant__ CUtensorMap tmap_w, const __grid_constant__ CUtensorMap tmap_x,
               const GemmParams p) {
    extern __shared__ __align__(1024) uint8_t smem_raw[];
    uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) &
                                               ~uintptr_t(1023));
    const int a_bytes = kBM * kBK * 2;
    const int b_bytes = p.b_bytes;
    const int stage_bytes = a_bytes + b_bytes;
    float* ep_stage = reinterpret_cast<float*>(smem + p.stages * stage_bytes);  // 4 x 16 x 36 floats
    uint64_t* full_bar = reinterpret_cast<uint64_t*>(ep_stage + 4 * 16 * kStageStride);
    uint64_t* empty_bar = full_bar + p.stages;
    uint64_t* tfull_bar = empty_bar + p.stages;  // [2]
    uint64_t* tempty_bar = tfull_bar + 2;        // [2]
    uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(tempty_bar + 2);
    float* rs = reinterpret_cast<float*>(reinterpret_cast<uint8_t*>(full_bar) + 256);  // [kRsFloats]

    const int warp = threadIdx.x >> 5;
    const int lane = threadIdx.x & 31;
    const int csize = CN * p.ks;
    const uint32_t crank = csize > 1 ? cluster_rank() : 0;
    const uint32_t rank = crank % CN;  // feature tile within the multicast pair
    const int kidx = int(crank) / CN;  // k share (k-split clusters)
    const int cluster = blockIdx.x / csize;

    if (warp == 0 && lane == 0) {
        tma_prefetch_desc(&tmap_w);
        tma_prefetch_desc(&tmap_x);
        for (int s = 0; s < p.stages; ++s) {
            mbar_init(&full_bar[s], 1);
            mbar_init(&empty_bar[s], TWO ? 1 : CN);
        }
        for (int a = 0; a < 2; ++a) {
            mbar_init(&tfull_bar[a], 1);
            mbar_init(&tempty_bar[a], TWO ? 8 : 4);  // 2-SM: both CTAs' epilogue warps
        }
        fence_mbar_init();
    }
    if (warp == 2) {
        if constexpr (TWO)
            tmem_alloc_2sm(tmem_slot, 512);
        else
            tmem_alloc(tmem_slot, 512);
    }
    tc_fence_before();
    __syncthreads();
    if (csize > 1) cluster_sync();  // remote barriers initialised before any multicast lands
    tc_fence_after();
    const uint32_t tmem_base = *tmem_slot;
    if (threadIdx.x == 0) GEMM_TRACE(0);
    pdl_launch_dependents();

    const int cl_tiles = p.m_tiles / CN;
    const bool leader = !TWO || rank == 0;

    if (warp == 3 && p.pf_kb > 0) {
        // L2 prefetch of this CTA's weight stream past what the smem pipeline loads up front:
        // independent of the previous kernel, so it is issued before griddepcontrol.wait and
        // streams while the previous kernel drains (its epilogue and tail leave HBM idle); the
        // main loop's TMA loads then hit L2. One contiguous run per weight row and segment.
        int skip = p.stages, budget = p.pf_kb;
        for_each_seg(p, cluster, kidx, [&](const Seg& w) {
            int kb = w.kb0;
            const int sk = min(skip, w.kb1 - kb);
            kb += sk;
            skip -= sk;
            const int n = min(budget, w.kb1 - kb);
            if (n <= 0) return;
            budget -= n;
            const int mt = tile_mtc(p, w.ut, cl_tiles) * CN + int(rank);
            for (int r = lane; r < kBM; r += 32)
                prefetch_l2_bulk(p.w + (size_t(mt) * kBM + r) * p.K + size_t(kb) * kBK, uint32_t(n * kBK * 2));
        });
    }
    if (p.rs_ssq && warp >= 3) {
        // RowNorm consumer: the RMSNorm scale of every token row from the producer's slice sums
        // of squares (parts summed in order: deterministic), by warps 3..7 while the producer
        // and MMA warps stream the first tiles; 32 loads per thread in flight
        pdl_wait();
        for (int t = int(threadIdx.x) - 96; t < p.T; t += kGemmThreads - 96) {
            float s = 0.f;
            for (int i0 = 0; i0 < p.rs_parts; i0 += 32) {
                float v[32];
#pragma unroll
                for (int k = 0; k < 32; ++k)
                    v[k] = i0 + k < p.rs_parts ? __ldcg(p.rs_ssq + size_t(i0 + k) * p.T + t) : 0.f;
#pragma unroll
                for (int k = 0; k < 32; ++k) s += v[k];
            }
            rs[t] = 1.0f / sqrtf(s / float(p.rs_d) + p.rs_eps);
            if (p.rs_out && blockIdx.x == 0) p.rs_out[t] = rs[t];
        }
        asm volatile("bar.sync 2, 160;" ::: "memory");  // warps 3..7: the scales are in smem
    }
    if (warp == 0) {
        if (elect_one()) {
            const uint64_t pol_w = policy_evict_first();
            const uint64_t pol_x = policy_evict_last();
            const uint16_t mask = uint16_t(((1u << CN) - 1) << (kidx * CN));
            // 2-SM: every TMA completes on the leader's full barrier, which expects both CTAs' bytes
            auto load_w = [&](int s, int kb, int mt) {
                if constexpr (TWO) {
                    if (leader) mbar_arrive_expect_tx(&full_bar[s], 2 * stage_bytes);
                    tma_load_2d_2sm(smem + s * stage_bytes, &tmap_w, mapa_shared(smem_u32(&full_bar[s]), 0),
                                    kb * kBK, mt * kBM, pol_w);
                } else {
                    mbar_arrive_expect_tx(&full_bar[s], stage_bytes);
                    tma_load_2d_hint(smem + s * stage_bytes, &tmap_w, &full_bar[s], kb * kBK, mt * kBM, pol_w);
                }
            };
            // weights first (independent of the previous kernel), activations after pdl_wait
            int pre = 0;
            for_each_seg(p, cluster, kidx, [&](const Seg& w) {
                const int mt = tile_mtc(p, w.ut, cl_tiles) * CN + int(rank);
                for (int kb = w.kb0; kb < w.kb1 && pre < p.stages; ++kb, ++pre) load_w(pre, kb, mt);
            });
            pdl_wait();
            int i = 0;
            for_each_seg(p, cluster, kidx, [&](const Seg& w) {
                const int tbk = tile_tbk(p, w.ut, cl_tiles);
                const int mt = tile_mtc(p, w.ut, cl_tiles) * CN + int(rank);
                for (int kb = w.kb0; kb < w.kb1; ++kb, ++i) {
                    const int s = i % p.stages;
                    const uint32_t round = i / p.stages;
                    uint8_t* sa = smem + s * stage_bytes;
                    uint8_t* sb = sa + a_bytes;
                    if (i >= pre) {
                        mbar_wait(&empty_bar[s], (round & 1) ^ 1);
                        load_w(s, kb, mt);
                    }
                    if constexpr (TWO) {
                        // this CTA's half of each instruction's token columns (<= 2 instructions)
                        const uint32_t lb = mapa_shared(smem_u32(&full_bar[s]), 0);
                        const int n0 = min(256, p.tb_pad);
                        tma_load_2d_2sm(sb, &tmap_x, lb, kb * kBK, tbk * p.tb + int(rank) * (n0 / 2), pol_x);
                        if (p.tb_pad > 256)
                            tma_load_2d_2sm(sb + 128 * 128, &tmap_x, lb, kb * kBK,
                                            tbk * p.tb + 256 + int(rank) * ((p.tb_pad - 256) / 2), pol_x);
                    } else if (CN > 1) {
                        tma_load_2d_mc(sb + rank * p.brows * kBK * 2, &tmap_x, &full_bar[s], kb * kBK,
                                       tbk * p.tb + int(rank) * p.brows, mask);
                    } else {
                        tma_load_2d(sb, &tmap_x, &full_bar[s], kb * kBK, tbk * p.tb);
                    }
                }
            });
            GEMM_TRACE(1);
            // drain: every stage released by every CTA (no remote arrival after we exit)
            const int n = i;
            for (int k = (n > p.stages ? n - p.stages : 0); k < n; ++k)
                mbar_wait(&empty_bar[k % p.stages], (uint32_t(k / p.stages) & 1));
        }
    } else if (warp == 1 && leader) {
        int i = 0, seg = 0;
        for_each_seg(p, cluster, kidx, [&](const Seg& w) {
            const int tbk = tile_tbk(p, w.ut, cl_tiles);
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
                        if constexpr (TWO) {
                            // fixed split of the padded token block (matches the producer's halves)
                            const int n_c = c == 0 ? min(256, p.tb_pad) : p.tb_pad - 256;
                            if (n_c <= 0) break;
                            const uint32_t idesc = umma_idesc_bf16(2 * kBM, n_c);
#pragma unroll
                            for (int k = 0; k < kBK / 16; ++k)
                                umma_bf16_2sm(acc + c * 256, umma_sdesc_sw128(sa + k * 32),
                                              umma_sdesc_sw128(sb + c * 128 * 128 + k * 32), idesc,
                                              (kb > w.kb0 || k > 0) ? 1u : 0u);
                        } else {
                            const int n_c = min(256, t_here - 256 * c);
                            if (n_c <= 0) break;
                            const uint32_t idesc = umma_idesc_bf16(kBM, (n_c + 15) & ~15);
#pragma unroll
                            for (int k = 0; k < kBK / 16; ++k)
                                umma_bf16(acc + c * 256, umma_sdesc_sw128(sa + k * 32),
                                          umma_sdesc_sw128(sb + c * 256 * 128 + k * 32), idesc,
                                          (kb > w.kb0 || k > 0) ? 1u : 0u);
                        }
                    }
                    if constexpr (TWO) {
                        umma_commit_2sm(&empty_bar[s], 0x3);
                        if (kb == w.kb1 - 1) umma_commit_2sm(&tfull_bar[a], 0x3);
                    } else {
                        if (CN > 1)
                            umma_commit_mc(&empty_bar[s], uint16_t(((1u << CN) - 1) << (kidx * CN)));
                        else
                            umma_commit(&empty_bar[s]);
                        if (kb == w.kb1 - 1) umma_commit(&tfull_bar[a]);
                    }
                }
                __syncwarp();
            }
            ++seg;
        });
        if (lane == 0) GEMM_TRACE(2);
    } else if (warp >= 4 && p.ks == 1) {
        pdl_wait();
        const int q = warp & 3;
        float* stage = ep_stage + q * 16 * kStageStride;
        volatile int* last_flag = reinterpret_cast<volatile int*>(tmem_slot + 1);
        const int row = lane >> 1, half = lane & 1;
        const size_t slot_elems = size_t(p.tb_pad) * kBM;
        int seg = 0;
        for_each_seg(p, cluster, kidx, [&](const Seg& w) {
            const int tbk = tile_tbk(p, w.ut, cl_tiles);
            const int mt = tile_mtc(p, w.ut, cl_tiles) * CN + int(rank);
            const int t0 = tbk * p.tb;
            const int t_here = min(p.tb, p.T - t0);
            const int a = seg % p.n_acc;
            const uint32_t acc = tmem_base + uint32_t(a * 256) + (uint32_t(q * 32) << 16);
            const int f_slice = mt * kBM + q * 32;
            mbar_wait(&tfull_bar[a], (seg / p.n_acc) & 1);
            tc_fence_after();
            float v[16];
            uint32_t r[16];
            if (w.kb0 == 0 && w.kb1 == p.KB) {  // whole tile: fused epilogue straight from TMEM
                for (int c0 = 0; c0 < t_here; c0 += 16) {
                    tmem_ld16(acc + c0, r);
                    tmem_ld_wait();
                    const bool ok = transpose16(stage, reinterpret_cast<float*>(r), lane, c0, t_here, v);
                    epi_store(p, v, ok, lane, t0 + c0 + row, f_slice, ok && p.rs_ssq ? rs[t0 + c0 + row] : 1.f);
                    if (p.ssq_out) {  // slice (tile, warp q) of token row t: lanes 2r, 2r+1
                        float ss = 0.f;
#pragma unroll
                        for (int j = 0; j < 16; ++j) {
                            const float xb = round_bf(v[j]);  // the stored bf16 of x
                            ss += xb * xb;
                        }
                        ss += __shfl_xor_sync(0xffffffffu, ss, 1);
                        if (ok && half == 0) rs[q * kMaxTB + c0 + row] = ss;  // smem [warp][row]
                    }
                }
                if (p.ssq_out) {  // the 4 warps' slices of each row, summed in warp order
                    epi_bar();
                    for (int i = int(threadIdx.x) - 128; i < t_here; i += 128)
                        p.ssq_out[size_t(mt) * p.T + t0 + i] =
                            ((rs[i] + rs[kMaxTB + i]) + rs[2 * kMaxTB + i]) + rs[3 * kMaxTB + i];
                    epi_bar();
                }
            } else {
                // split tile: park this piece (TMEM-native layout [chunk][feature][16 tokens]: each
                // thread stores / loads its own 64 contiguous bytes), count the arrival; the last
                // arriver sums all pieces in k order (deterministic) and runs the epilogue.
                if (p.planes) {  // narrow GEMM: fp32 partial into plane (k range) [T][N]
                    float* plane = p.slots + size_t(cluster % p.planes) * p.T * p.N;
                    for (int c0 = 0; c0 < t_here; c0 += 16) {
                        tmem_ld16(acc + c0, r);
                        tmem_ld_wait();
                        if (transpose16(stage, reinterpret_cast<float*>(r), lane, c0, t_here, v)) {
                            float4* dst = reinterpret_cast<float4*>(plane + size_t(t0 + c0 + row) * p.N +
                                                                    f_slice + half * 16);
#pragma unroll
                            for (int i = 0; i < 4; ++i)
                                __stcg(dst + i, make_float4(v[4 * i], v[4 * i + 1], v[4 * i + 2], v[4 * i + 3]));
                        }
                    }
                    goto seg_done;  // planes summed by splitk_reduce_kernel
                }
                const size_t fo = size_t(q * 32 + lane) * 16;
                const int n_chunks = (t_here + 15) / 16;
                float* mine = p.slots + ((size_t(cluster) * 2 + w.which) * CN + rank) * slot_elems;
                for (int ch = 0; ch < n_chunks; ++ch) {
                    tmem_ld16(acc + ch * 16, r);
                    tmem_ld_wait();
                    float4* dst = reinterpret_cast<float4*>(mine + size_t(ch) * kBM * 16 + fo);
#pragma unroll
                    for (int i = 0; i < 4; ++i)
                        __stcg(dst + i, make_float4(__uint_as_float(r[4 * i]), __uint_as_float(r[4 * i + 1]),
                                                    __uint_as_float(r[4 * i + 2]), __uint_as_float(r[4 * i + 3])));
                }
                if (p.defer) goto seg_done;  // pieces summed by splitk_finish_kernel
                __threadfence();
                epi_bar();
                const int tile_g0 = w.ut * p.KB;
                const int c_lo = sk_owner(p, tile_g0), c_hi = sk_owner(p, tile_g0 + p.KB - 1);
                if (threadIdx.x == 128) {
                    int* cnt = p.counters + size_t(w.ut) * CN + rank;
                    const int old = atomicAdd(cnt, 1);
                    const int last = old == c_hi - c_lo;
                    if (last) *cnt = 0;  // ready for the next launch
                    *last_flag = last;
                }
                epi_bar();
                const bool last = *last_flag != 0;
                epi_bar();  // flag read by all before the next segment rewrites it
                if (last) {
                    __threadfence();
                    for (int ch = 0; ch < n_chunks; ++ch) {
                        float own[16], sum[16];
                        tmem_ld16(acc + ch * 16, reinterpret_cast<uint32_t*>(own));
                        tmem_ld_wait();
                        sum_pieces(p, CN, rank, tile_g0, c_lo, c_hi, size_t(ch) * kBM * 16 + fo, cluster,
                                   own, sum);
                        const bool ok = transpose16(stage, sum, lane, ch * 16, t_here, v);
                        epi_store(p, v, ok, lane, t0 + ch * 16 + row, f_slice,
                                  ok && p.rs_ssq ? rs[t0 + ch * 16 + row] : 1.f);
                    }
                }
            }
        seg_done:
            tc_fence_before();
            __syncwarp();
            if (lane == 0) {
                if constexpr (TWO)
                    mbar_arrive_remote(mapa_shared(smem_u32(&tempty_bar[a]), 0));  // leader's MMA
                else
                    mbar_arrive(&tempty_bar[a]);
            }
            ++seg;
        });
        if (threadIdx.x == 128) GEMM_TRACE(3);
    }
    __syncthreads();
    if (p.ks > 1) {
        pdl_wait();
        mbar_wait(&tfull_bar[0], 0);
        tc_fence_after();
        if (threadIdx.x == 128) GEMM_TRACE(4);  // accumulator complete
        if (p.ks_push)
            ksplit_epilogue_push<CN>(p, smem, tmem_base, cluster, kidx, int(rank), warp, lane);
        else
            ksplit_epilogue<CN>(p, smem, tmem_base, cluster, kidx, int(rank), warp, lane, rs);
        tc_fence_before();
        if (threadIdx.x == 128) GEMM_TRACE(3);
    }
    if (csize > 1) cluster_sync();
    if (threadIdx.x == 0) GEMM_TRACE(5);
    if (warp == 2) {
        tc_fence_after();
        if constexpr (TWO)
            tmem_dealloc_2sm(tmem_base, 512);
        else
            tmem_dealloc(tmem_base, 512);
    }
}

// Deferred stream-K finish: block = (split tile, CTA rank, 16-token chunk); sums the tile's pieces
// in k order (same order as the in-kernel last arriver) and applies the fused epilogue. Spreads
// the reduction of narrow GEMMs (every tile split) over all SMs.
template <int CN>
__global__ void __launch_bounds__(128) splitk_finish_kernel(const GemmParams p) {
    pdl_launch_dependents();
    pdl_wait();
    __shared__ float stage_all[4][16 * kStageStride];
    const int n_chunks = (p.tb + 15) / 16;
    const int ch = blockIdx.x % n_chunks;
    const int rank = (blockIdx.x / n_chunks) % CN;
    const int ut = blockIdx.x / (n_chunks * CN);
    const int cl_tiles = p.m_tiles / CN;
    const int tbk = tile_tbk(p, ut, cl_tiles);
    const int mt = tile_mtc(p, ut, cl_tiles) * CN + rank;
    const int t0 = tbk * p.tb;
    const int t_here = min(p.tb, p.T - t0);
    if (ch * 16 >= t_here) return;
    const int q = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int tile_g0 = ut * p.KB;
    const int c_lo = sk_owner(p, tile_g0), c_hi = sk_owner(p, tile_g0 + p.KB - 1);
    if (c_lo == c_hi) return;  // one cluster covered the whole tile and finished it in-kernel
    float sum[16], v[16];
    sum_pieces(p, CN, rank, tile_g0, c_lo, c_hi, size_t(ch) * kBM * 16 + size_t(q * 32 + lane) * 16, -1,
               nullptr, sum);
    const bool ok = transpose16(stage_all[q], sum, lane, ch * 16, t_here, v);
    epi_store(p, v, ok, lane, t0 + ch * 16 + (lane >> 1), mt * kBM + q * 32);
}

// Narrow-GEMM reduction: the k-range planes summed in order (deterministic) + the fused epilogue,
// grid-stride over float4s of [T][N] (no shared memory: co-resides with the GEMM CTAs and waits
// at griddepcontrol.wait, so it runs the moment the GEMM retires).
__global__ void __launch_bounds__(256) splitk_reduce_kernel(const GemmParams p) {
    pdl_launch_dependents();
    pdl_wait();
    const size_t total = size_t(p.T) * p.N / 4;
    const size_t plane = size_t(p.T) * p.N;
    for (size_t i = blockIdx.x * size_t(blockDim.x) + threadIdx.x; i < total;
         i += size_t(gridDim.x) * blockDim.x) {
        float4 a = __ldcg(reinterpret_cast<const float4*>(p.slots) + i);
        for (int k = 1; k < p.planes; ++k) {
            const float4 b = __ldcg(reinterpret_cast<const float4*>(p.slots + k * plane) + i);
            a.x += b.x;
            a.y += b.y;
            a.z += b.z;
            a.w += b.w;
        }
        const size_t o = i * 4;
        if (p.epi == EPI_F32) {
            reinterpret_cast<float4*>(p.out_f32)[i] = a;
            continue;
        }
        if (p.epi == EPI_SILU) {  // gate columns pair with the up columns 16 further on
            const int c = int(o % p.N);
            if (c % 32 >= 16) continue;
            float4 u = __ldcg(reinterpret_cast<const float4*>(p.slots) + i + 4);
            for (int k = 1; k < p.planes; ++k) {
                const float4 b = __ldcg(reinterpret_cast<const float4*>(p.slots + k * plane) + i + 4);
                u.x += b.x;
                u.y += b.y;
                u.z += b.z;
                u.w += b.w;
            }
            const float g4[4] = {a.x, a.y, a.z, a.w}, u4[4] = {u.x, u.y, u.z, u.w};
            float h[4];
#pragma unroll
            for (int j = 0; j < 4; ++j) {
                const float gb = round_bf(g4[j]);
                h[j] = round_bf(__fdividef(gb, 1.0f + __expf(-gb))) * round_bf(u4[j]);
            }
            uint2 hv;
            hv.x = pack2(h[0], h[1]);
            hv.y = pack2(h[2], h[3]);
            const size_t t = o / p.N;
            *reinterpret_cast<uint2*>(p.out_bf16 + t * (p.N / 2) + (c / 32) * 16 + c % 32) = hv;
            continue;
        }
        float v[4] = {a.x, a.y, a.z, a.w};
        if (p.epi == EPI_RESID) {
            const uint2 rv = *reinterpret_cast<const uint2*>(p.resid + o);
            const __nv_bfloat162* rh = reinterpret_cast<const __nv_bfloat162*>(&rv);
            const float2 r0 = __bfloat1622float2(rh[0]), r1 = __bfloat1622float2(rh[1]);
            v[0] = r0.x + round_bf(v[0]);
            v[1] = r0.y + round_bf(v[1]);
            v[2] = r1.x + round_bf(v[2]);
            v[3] = r1.y + round_bf(v[3]);
        }
        uint2 ov;
        ov.x = pack2(v[0], v[1]);
        ov.y = pack2(v[2], v[3]);
        *reinterpret_cast<uint2*>(p.out_bf16 + o) = ov;
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

int make_tmap_3d_bf16(void* tmap_out, const void* base, uint64_t d0, uint64_t d1, uint64_t d2,
                      uint32_t b0, uint32_t b1, uint32_t b2) {
    auto fn = get_encode_fn();
    if (!fn) return -1;
    CUtensorMap* m = reinterpret_cast<CUtensorMap*>(tmap_out);
    cuuint64_t dims[3] = {d0, d1, d2};
    cuuint64_t strides[2] = {d0 * 2, d0 * d1 * 2};
    cuuint32_t box[3] = {b0, b1, b2};
    cuuint32_t estr[3] = {1, 1, 1};
    CUresult r = fn(m, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 3, const_cast<void*>(base), dims, strides, box,
                    estr, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                    CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    return r == CUDA_SUCCESS ? 0 : -2;
}

size_t gemm_workspace_floats() { return kWorkspaceFloats; }

static int pick_cn(int N) {
    static const int cn_env = getenv("DS_GEMM_CN") ? atoi(getenv("DS_GEMM_CN")) : 2;
    return (cn_env == 1 || (N / kBM) % 2 != 0) ? 1 : 2;
}

static GemmParams plan_gemm(int T, int N, int K, int max_clusters, int* cn_out);

int gemm_launch_count(int T, int N, int K, bool deferred) {
    int cn = 0;
    const GemmParams p = plan_gemm(T, N, K, 0, &cn);
    return 1 + ((p.defer && !(deferred && p.planes)) ? 1 : 0);
}

// Token block `tb` with `cn` CTAs per cluster: padding, TMA box, shared-memory stage and depth.
static bool set_block(GemmParams& p, int tb, int cn) {
    static const int two_sm_env = getenv("DS_GEMM_2SM") ? atoi(getenv("DS_GEMM_2SM")) : 1;
    p.tb = tb;
    p.t_blocks = (p.T + tb - 1) / tb;
    p.tb_pad = (tb + 15) & ~15;
    p.brows = p.tb_pad / cn;
    p.b_bytes = p.tb_pad * kBK * 2;
    p.two_sm = 0;
    if (cn == 2 && two_sm_env) {  // 2-SM MMA: half of each instruction's tokens per CTA
        p.two_sm = 1;
        p.brows = p.tb_pad <= 256 ? p.tb_pad / 2 : 128;
        p.b_bytes = p.tb_pad <= 256 ? p.tb_pad / 2 * 128 : 2 * 128 * 128;
    }
    const int stage_bytes = kBM * kBK * 2 + p.b_bytes;
    p.stages = std::min(12, (kSmemBudget - kFixedSmem) / stage_bytes);
    p.n_acc = p.tb_pad <= 256 ? 2 : 1;
    return p.stages >= 2 && p.brows <= 256;
}

// Tile shape, pipeline depth and the work partition of one GEMM (a negative p.T is the error code
// of an unsupported shape). Modes, by how many 128-feature tiles there are per SM:
//  * wide (>= one wave of tiles): whole tiles data-parallel, the remainder wave stream-K split
//    (<= 128 tokens, last-arriver fixup) or whole;
//  * very narrow, <= 256 tokens (o / down at 8B): K split 4 ways inside 4-CTA clusters reduced
//    through distributed shared memory;
//  * narrow with >= 64 tokens per block: token blocks split instead of K (no partial sums; the
//    blocks sharing a weight tile stream it at the same time, L2 serves the re-reads);
//  * otherwise: K split into planes summed by the consumer kernel (or a reduction kernel).
static GemmParams plan_gemm(int T, int N, int K, int max_clusters, int* cn_out) {
    GemmParams p{};
    int cn = pick_cn(N);
    p.T = T;
    p.N = N;
    p.K = K;
    if (K % kBK != 0 || N % kBM != 0) { p.T = -3; return p; }
    p.m_tiles = N / kBM;
    p.KB = K / kBK;
    p.ks = 1;
    // Token block: <= 512 (the TMEM columns); above `tb_max` tokens the blocks shrink to 256
    // (double-buffered accumulators: the epilogue overlaps the next tile) and run token-block-
    // fastest so the blocks sharing a weight tile stream it concurrently (L2 serves the re-reads).
    static const int tb_max = getenv("DS_GEMM_TB_MAX") ? atoi(getenv("DS_GEMM_TB_MAX")) : kMaxTB;
    int tb0 = T < kMaxTB ? T : kMaxTB;
    if (T > tb_max) {
        tb0 = std::min(tb0, 256);
        p.tb_fast = 1;
    }
    if (cn == 1 && (tb0 + 15) / 16 * 16 > 256) cn = (p.m_tiles % 2 == 0) ? 2 : 1;  // TMA box <= 256
    if (!set_block(p, tb0, cn)) { p.T = cn == 1 ? -9 : -4; return p; }
    int nc = kNumSMs / cn;
    if (max_clusters > 0 && nc > max_clusters) nc = max_clusters;
    const int cl_tiles = p.m_tiles / cn;
    int tiles = p.t_blocks * cl_tiles;

    static const int ksplit_env = getenv("DS_GEMM_KSPLIT") ? atoi(getenv("DS_GEMM_KSPLIT")) : 1;
    static const int ts_min = getenv("DS_GEMM_TS_MIN") ? atoi(getenv("DS_GEMM_TS_MIN")) : 257;
    const int tiles1 = p.t_blocks * p.m_tiles;
    static const int ks2_env = getenv("DS_GEMM_KS2") ? atoi(getenv("DS_GEMM_KS2")) : 0;
    // DS_GEMM_KS3=1: 3-way k-split clusters where 3 * tiles fill the SMs (q/k/v at 8B: 144 CTAs)
    static const int ks3_env = getenv("DS_GEMM_KS3") ? atoi(getenv("DS_GEMM_KS3")) : 0;
    const int ks_pick = kNumSMs / tiles1 >= 4   ? 4
                        : (ks3_env && kNumSMs / tiles1 >= 3) ? 3
                        : (ks2_env && kNumSMs / tiles1 >= 2) ? 2
                                                              : 1;
    if (ksplit_env && max_clusters <= 0 && p.tb_pad <= 256 && p.KB >= 8 && ks_pick > 1 &&
        T < ts_min) {
        GemmParams q = p;
        if (set_block(q, p.tb, 1) && size_t(q.stages) * (kBM * kBK * 2 + q.b_bytes) >= size_t(q.tb_pad) * kBM * 4) {
            q.ks = ks_pick;
            q.n_clusters = tiles1;
            *cn_out = 1;
            return q;
        }
    }
    // (weights must stay L2-resident across the concurrent blocks: measured at T = 320..456,
    // q/k/v 50 MB and o 32 MB gain 25-30%, down 117 MB loses 25%; below 257 tokens the k-split
    // cluster / plane modes win)
    if (tiles < nc && max_clusters <= 0 && T >= ts_min && T >= 128 &&
        size_t(N) * K * 2 <= (size_t(64) << 20)) {
        // token split: s blocks of >= 64 tokens per weight tile, at most one wave of tiles
        const int s_t = std::min(nc / cl_tiles, T / 64);
        if (s_t >= 2) {
            GemmParams q = p;
            const int tb = std::min(kMaxTB, ((T + s_t - 1) / s_t + 15) / 16 * 16);
            if (set_block(q, tb, cn)) {
                q.tb_fast = 1;
                q.n_clusters = q.t_blocks * cl_tiles;
                q.dp_rounds = 1;
                *cn_out = cn;
                return q;
            }
        }
    }
    // whole waves data-parallel, the remainder stream-K over all clusters
    p.n_clusters = std::min(nc, tiles * p.KB);
    p.dp_rounds = tiles / p.n_clusters;
    p.sk_tiles = tiles - p.dp_rounds * p.n_clusters;
    p.n_sk = std::min(p.n_clusters, p.sk_tiles * p.KB);
    if (p.dp_rounds == 0 && p.sk_tiles * 2 > p.n_sk) {
        // more than half a wave of tiles: run them whole (one round), no partial sums
        p.n_clusters = p.sk_tiles;
        p.dp_rounds = 1;
        p.sk_tiles = p.n_sk = 0;
    }
    if (p.dp_rounds == 0 && p.sk_tiles * 2 <= p.n_sk) {
        // narrow GEMM: every tile split into the same number of k ranges, one piece per cluster
        // (no range straddles two tiles: half the pieces of a free partition, a few idle SMs)
        p.n_sk = p.sk_tiles * std::min(p.n_sk / p.sk_tiles, p.KB);
        p.n_clusters = p.n_sk;
        // one plane per k range while they fit the workspace (else TMEM-layout pieces)
        if (size_t(p.n_sk / p.sk_tiles) * T * N + T <= kWorkspaceFloats - kCounterInts)
            p.planes = p.n_sk / p.sk_tiles;
    }
    // Remainder tiles run whole (n_sk = sk_tiles: one whole tile per remainder cluster) above
    // 128 tokens: half the SMs still saturate HBM in the last round, while the last arriver's
    // piece reads delay its next epilogue (measured at T = 180 / 256: 49 / 55 us whole vs 55 / 64
    // stream-K); at <= 128 tokens stream-K balancing wins (e.g. 40.9 vs 44.0 us at T = 16).
    static const int whole_env = getenv("DS_GEMM_WHOLE") ? atoi(getenv("DS_GEMM_WHOLE")) : -1;
    const bool whole = whole_env >= 0 ? whole_env != 0 : p.tb_pad > 128;
    if (p.dp_rounds > 0 && whole) p.n_sk = p.sk_tiles;
    // Pieces per stream-K remainder tile (DS_GEMM_SKP; 0 = as many as clusters): a tile split
    // over many clusters makes its last arriver read every other piece's partial sums before
    // its data-parallel tiles. 70B gate/up (224 pair tiles: 3 rounds + 2 remainder tiles over 74
    // clusters, 37 pieces each) at T = 49: 188 us uncapped, 153 / 148 / 146 us with 2 / 4 / 8
    // pieces, 155 us with 16; T = 128: 225 -> 151 us; 8B gate/up and the LM head unchanged
    // (their remainders already split in <= 2). Measured twice: profiles/r02_gemm_skp.txt.
    // (Capped stream-K remainders above 128 tokens instead of whole tiles: faster for 70B gate/up
    // at T = 160-256, slower on the 8B and prefill shapes -- not adopted.)
    static const int skp = getenv("DS_GEMM_SKP") ? atoi(getenv("DS_GEMM_SKP")) : kSkPieces;
    if (p.dp_rounds > 0 && !whole && skp > 0 && p.sk_tiles > 0)
        p.n_sk = std::min(p.n_sk, p.sk_tiles * skp);
    // the in-kernel last arriver pays off when its reads overlap the next tile's MMAs (data-
    // parallel tiles follow, accumulator double-buffered); otherwise a finish kernel spreads them
    p.defer = (p.sk_tiles > 0 && p.dp_rounds == 0) ? 1 : 0;
    *cn_out = cn;
    return p;
}

// A consumer row scale is applied wherever the output is finished: the kernel's epilogues (whole
// tiles, the stream-K last arriver, k-split pull) or the consumer of deferred planes — not the
// separate reduction / finish kernels, and for at most kRsMax rows (shared-memory scales).
static bool rowscale_ok(const GemmParams& p, int T, bool deferred) {
    if (p.T < 0 || T > kRsMax || p.ks_push) return false;
    if (p.planes) return deferred;
    return !p.defer;
}

int gemm_describe(int T, int N, int K, int32_t* out) {
    int cn = 0;
    const GemmParams p = plan_gemm(T, N, K, 0, &cn);
    const int32_t v[12] = {p.T < 0 ? p.T : 0, cn, p.n_clusters, p.dp_rounds, p.sk_tiles, p.n_sk, p.ks,
                           p.planes, p.defer, p.tb, p.t_blocks, p.KB};
    for (int i = 0; i < 12; ++i) out[i] = v[i];
    return p.T < 0 ? p.T : 0;
}

bool gemm_rowscale_ok(int T, int N, int K, bool deferred) {
    int cn = 0;
    GemmParams p = plan_gemm(T, N, K, 0, &cn);
    static const int push_env = getenv("DS_GEMM_KSPUSH") ? atoi(getenv("DS_GEMM_KSPUSH")) : 0;
    p.ks_push = (push_env && p.ks > 1 &&
                 ksplit_push_smem(p.ks) <= size_t(p.stages) * size_t(kBM * kBK * 2 + p.b_bytes)) ? 1 : 0;
    return rowscale_ok(p, T, deferred);
}

int gemm_bf16(const GemmWeight& w, const __nv_bfloat16* x, int T, int epi, __nv_bfloat16* out_bf16,
              const __nv_bfloat16* resid, float* out_f32, float* workspace, size_t workspace_floats,
              int max_clusters, cudaStream_t stream, Planes* defer, const RowNorm* rn, int* ssq_parts) {
    const int N = w.N, K = w.K;
    if (defer) *defer = Planes{};
    if (ssq_parts) *ssq_parts = 0;
    if (T <= 0) return 0;
    int cn = 1;
    GemmParams p = plan_gemm(T, N, K, max_clusters, &cn);
    if (p.T < 0) return p.T;
    const int tiles = p.t_blocks * (p.m_tiles / cn);
    const int stage_bytes = kBM * kBK * 2 + p.b_bytes;
    const int fixed = kFixedSmem;
    // workspace: [counters: kCounterInts, shared by every shape: a launch leaves them all 0]
    //            [slots: n_clusters * 2 * cn * tb_pad * 128 floats]
    const size_t n_cnt = kCounterInts;
    const size_t need = n_cnt + (p.planes ? size_t(p.planes) * T * N + T
                                          : size_t(p.n_clusters) * 2 * cn * p.tb_pad * kBM);
    if (p.sk_tiles > 0 && (!workspace || workspace_floats < need || size_t(tiles) * cn > n_cnt))
        return -7;
    p.epi = epi;
    p.out_bf16 = out_bf16;
    p.resid = resid;
    p.out_f32 = out_f32;
    p.counters = reinterpret_cast<int*>(workspace);
    p.slots = workspace + n_cnt;
    p.trace = g_gemm_trace;
    p.w = w.data;
    {   // L2 prefetch budget (DS_GEMM_L2PF=MB: a weight matrix up to 64 MB entirely, else this
        // many MB over the CTAs). Off: measured slower on every 8B shape (qkv 20.7 -> 22.4 us,
        // down 30.8 -> 33.6 us at T = 180) and 14.13 k -> 13.69 k tok/s on config 2
        // (profiles/r02_ab_l2pf.txt): the prefetch competes with the previous kernel's stream.
        // DS_GEMM_L2PF_KMIN restricts it to GEMMs with K >= the value (the down projection, whose
        // CTAs start on the SMs gate/up's last round leaves idle): slower too
        // (profiles/r02_ab_l2pf_down.txt).
        static const int pf_env = getenv("DS_GEMM_L2PF") ? atoi(getenv("DS_GEMM_L2PF")) : 0;
        static const int pf_kmin = getenv("DS_GEMM_L2PF_KMIN") ? atoi(getenv("DS_GEMM_L2PF_KMIN")) : 0;
        const size_t wbytes = size_t(N) * K * 2;
        const int ctas = p.n_clusters * cn * p.ks;
        const size_t per_kb = size_t(kBM) * kBK * 2;  // one k-block of one CTA's 128 rows
        if (pf_env <= 0 || ctas <= 0 || K < pf_kmin)
            p.pf_kb = 0;
        else if (wbytes <= (size_t(64) << 20))
            p.pf_kb = 1 << 20;
        else
            p.pf_kb = int((size_t(pf_env) << 20) / size_t(ctas) / per_kb);
    }
    {   // k-split epilogue: push form when the parked window + receive blocks fit the pipeline
        // shared memory (DS_GEMM_KSPUSH=1). Off by default: measured slower than the pull form
        // (o at T = 180: 18.9 vs 15.3-15.9 us per launch, profiles/r02_gemm_trace_push.txt)
        static const int push_env = getenv("DS_GEMM_KSPUSH") ? atoi(getenv("DS_GEMM_KSPUSH")) : 0;
        p.ks_push = (push_env && p.ks > 1 &&
                     ksplit_push_smem(p.ks) <= size_t(p.stages) * size_t(kBM * kBK * 2 + p.b_bytes)) ? 1 : 0;
    }
    if (rn && rn->ssq_out && epi == EPI_RESID && T <= rn->max_rows) {
        // RowNorm producer: only where every output row slice is final inside this kernel
        // (k-split clusters with the pull epilogue, or whole tiles: no stream-K pieces, no planes)
        const bool whole = p.ks == 1 && !p.planes && !p.defer && (p.sk_tiles == 0 || p.n_sk == p.sk_tiles);
        const bool ksplit = p.ks > 1 && !p.ks_push;
        if (whole || ksplit) {
            p.ssq_out = rn->ssq_out;
            if (ssq_parts) *ssq_parts = p.m_tiles;  // one slice per 128-feature tile
        }
    }
    if (rn && rn->ssq_in) {  // RowNorm consumer (the caller checked gemm_rowscale_ok)
        if (!rowscale_ok(p, T, defer != nullptr) || p.ssq_out) return -8;
        p.rs_ssq = rn->ssq_in;
        p.rs_parts = rn->parts;
        p.rs_d = rn->d;
        p.rs_eps = rn->eps;
        if (p.planes) p.rs_out = p.slots + size_t(p.planes) * T * N;  // behind the planes
    }
    alignas(64) CUtensorMap tx;
    if (make_tmap_2d_bf16(&tx, x, T, K, p.brows, kBK) != 0) return -5;
    const size_t smem = size_t(p.stages) * stage_bytes + fixed;
    cudaLaunchConfig_t cfg{};
    cfg.gridDim = dim3(p.n_clusters * cn * p.ks);
    cfg.blockDim = dim3(kGemmThreads);
    cfg.dynamicSmemBytes = smem;
    cfg.stream = stream;
    cudaLaunchAttribute attr[2];
    attr[0].id = cudaLaunchAttributeClusterDimension;
    attr[0].val.clusterDim.x = cn * p.ks;
    attr[0].val.clusterDim.y = 1;
    attr[0].val.clusterDim.z = 1;
    attr[1].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[1].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 2;
    const CUtensorMap& tw = *reinterpret_cast<const CUtensorMap*>(w.tmap);
    cudaError_t e = p.two_sm ? cudaLaunchKernelEx(&cfg, gemm_tc_kernel<2, true>, tw, tx, p)
                    : cn == 2 ? cudaLaunchKernelEx(&cfg, gemm_tc_kernel<2, false>, tw, tx, p)
                              : cudaLaunchKernelEx(&cfg, gemm_tc_kernel<1, false>, tw, tx, p);
    if (e != cudaSuccess) return -6;
    static const bool no_finish = getenv("DS_GEMM_NOFINISH") != nullptr;  // debug: timing only
    if (p.planes && defer) {
        defer->p = p.slots;
        defer->n = p.planes;
        defer->stride = size_t(T) * N;
        if (p.rs_ssq) defer->rs = p.rs_out;  // the consumer of the planes applies the row scales
    } else if (p.planes && !no_finish) {
        const size_t total4 = size_t(T) * N / 4;
        const int blocks = int(std::min<size_t>((total4 + 255) / 256, size_t(kNumSMs) * 8));
        e = launch_pdl(splitk_reduce_kernel, dim3(blocks), dim3(256), 0, stream, p);
        if (e != cudaSuccess) return -6;
    } else if (p.defer && !no_finish) {
        const dim3 grid(p.sk_tiles * cn * ((p.tb + 15) / 16));
        e = cn == 2 ? launch_pdl(splitk_finish_kernel<2>, grid, dim3(128), 0, stream, p)
                    : launch_pdl(splitk_finish_kernel<1>, grid, dim3(128), 0, stream, p);
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
    cudaFuncGetAttributes(&a, gemm_tc_kernel<1, false>);
    cudaFuncGetAttributes(&a, gemm_tc_kernel<2, false>);
    cudaFuncGetAttributes(&a, gemm_tc_kernel<2, true>);
    cudaFuncGetAttributes(&a, splitk_reduce_kernel);
    cudaFuncGetAttributes(&a, splitk_finish_kernel<1>);
    cudaFuncGetAttributes(&a, splitk_finish_kernel<2>);
    cudaFuncSetAttribute(gemm_tc_kernel<1, false>, cudaFuncAttributeMaxDynamicSharedMemorySize, kSmemBudget + 2048);
    cudaFuncSetAttribute(gemm_tc_kernel<2, false>, cudaFuncAttributeMaxDynamicSharedMemorySize, kSmemBudget + 2048);
    cudaFuncSetAttribute(gemm_tc_kernel<2, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, kSmemBudget + 2048);
}

}  // namespace ds
