// Launchers for the sm_100a stage-forward kernels (host-callable, stream-ordered).
#pragma once

#include <cuda_bf16.h>
#include <cuda_runtime.h>
#include <stddef.h>
#include <stdint.h>

#include "common.cuh"

namespace ds {

enum GemmEpilogue : int {
    EPI_BF16 = 0,     // out = bf16(acc)
    EPI_RESID = 1,    // out = bf16(resid + bf16(acc))   (residual add fused; out may alias resid)
    EPI_F32 = 2,      // out = acc (fp32, logits)
    EPI_SILU = 3,     // gate/up GEMM (16-row interleaved weight): out[t, N/2] =
                      //   bf16(bf16(silu(bf16(gate))) * bf16(up))
};

// A weight matrix [N, K] (row-major, K contiguous) with its TMA descriptor.
struct GemmWeight {
    const __nv_bfloat16* data = nullptr;
    int N = 0, K = 0;
    alignas(64) unsigned char tmap[128];
};

// Split-K partial planes a narrow GEMM leaves for its consumer kernel to sum (in plane order,
// then the GEMM's epilogue rounding) instead of a separate reduction: plane k of row t, column
// c is p[k * stride + t * ld + c]. n == 0: no planes, the GEMM wrote its final output.
struct Planes {
    const float* p = nullptr;
    int n = 0;
    size_t stride = 0;
    // RowNorm consumer deferred with the planes: row t of the sum is scaled by rs[t] (the
    // GEMM's row scales) before rounding; nullptr: no scale
    const float* rs = nullptr;
};

// RMSNorm split across a residual GEMM and the GEMM that consumes the normalised rows (unit
// gains): the producer (EPI_RESID, out = x) writes the sums of squares of its output row slices
// (ssq_out[part][t], parts returned through ssq_parts: no atomics, no extra pass); the consumer
// reads x itself and scales its output row t by r[t] = 1 / sqrt(sum of the parts / d + eps):
// out = bf16(r[t] * sum_k x[t, k] W[n, k]) instead of the GEMM of bf16(x[t] * r[t]).
struct RowNorm {
    float* ssq_out = nullptr;  // producer side (>= (N / 128) * T floats)
    int max_rows = 0;
    const float* ssq_in = nullptr;  // consumer side
    int parts = 0, d = 0;
    float eps = 0.f;
};

int gemm_weight_init(GemmWeight* w, const __nv_bfloat16* data, int N, int K);
// Stream-K pieces + per-tile arrival counters; allocate once, zero-initialised, one per stream.
size_t gemm_workspace_floats();
// Debug: per-CTA phase timestamps (globaltimer ns, 8 slots per CTA) for subsequent launches.
void gemm_set_trace(unsigned long long* device_buf);
// Kernel launches gemm_bf16 issues for a shape (2 with a reduction / finish kernel; `deferred`:
// called with a Planes out-parameter).
int gemm_launch_count(int T, int N, int K, bool deferred = false);
// out[T, N] = epi(X[T, K] . W[N, K]^T). max_clusters > 0 caps the 2-CTA clusters (tests use it
// to force other data-parallel / stream-K partitions); 0 = all SMs.
// With `defer` != nullptr, a GEMM that would end in the split-K reduction kernel instead leaves
// its planes in the workspace and describes them in *defer (the consumer kernel finishes it);
// otherwise *defer = {} and the output is final.
// RowNorm: as producer (rn->ssq_out, EPI_RESID) the GEMM writes the slice sums of squares when
// its partition finishes whole rows in-kernel (k-split clusters or whole tiles) and returns the
// part count in *ssq_parts (0: not written, the caller normalises with rmsnorm_rows); as consumer
// (rn->ssq_in) it scales its output rows — only where gemm_rowscale_ok (returns -8 otherwise).
int gemm_bf16(const GemmWeight& w, const __nv_bfloat16* x, int T, int epi, __nv_bfloat16* out_bf16,
              const __nv_bfloat16* resid, float* out_f32, float* workspace, size_t workspace_floats,
              int max_clusters, cudaStream_t stream, Planes* defer = nullptr,
              const RowNorm* rn = nullptr, int* ssq_parts = nullptr);
bool gemm_rowscale_ok(int T, int N, int K, bool deferred);
// The work partition plan_gemm picks (host arithmetic only, no device): out[12] = {status, CTAs
// per cluster, clusters, data-parallel rounds, stream-K tiles, stream-K clusters, k-split ways,
// planes, deferred finish, tokens per block, token blocks, k-blocks per tile}.
int gemm_describe(int T, int N, int K, int32_t* out);

// Counter-based weight init (bf16(uniform(-1,1) * scale)); see oracle/llama_ref.c ds_ref_weight.
// interleave_part >= 0 writes the [rows, cols] tensor into the gate/up interleaved layout:
// canonical row r of tensor `part` (0 gate, 1 up) lands at row 32*(r/16) + 16*part + r%16, so a
// 32-row TMEM slice holds 16 gate and the matching 16 up features (EPI_SILU).
void init_weights(__nv_bfloat16* dst, uint64_t seed, uint64_t tensor_id, int64_t rows, int64_t cols,
                  float scale, int interleave_part, cudaStream_t stream);
void fill_bf16(__nv_bfloat16* dst, int64_t n, float v, cudaStream_t stream);

// x[t] = E[token[t]]; tokens come from prompt ids or from last_token[req] for decode rows.
void embed_rows(const __nv_bfloat16* emb, const int32_t* tokens, int T, int d, __nv_bfloat16* x,
                cudaStream_t stream);
// y[i] = bf16(g * bf16(x[row_i] * rsqrt(mean(x^2) + eps))); rows = index list or identity.
// With pending planes (identity rows only): first x[i] = bf16(x[i] + bf16(sum of planes)) (the
// deferred residual GEMM epilogue), written back to x; y == nullptr skips the normalisation.
void rmsnorm_rows(const __nv_bfloat16* x, const int32_t* rows, int n_rows, int d,
                  const __nv_bfloat16* g, float eps, __nv_bfloat16* y, cudaStream_t stream,
                  const Planes& pending = Planes{});

struct KvLayout {
    __nv_bfloat16* pool = nullptr;  // [n_pages][L_stage][2][n_kv][256][d_head]
    int64_t page_elems = 0;
    int n_layers = 0, n_kv = 0, d_head = 0;
    // TMA view of the pool (host copy of a CUtensorMap, 128-byte aligned): rows of d_head
    // elements, row = ((page * L + layer) * 2 + K|V) * n_kv + kv head) * 256 + token; 16-row x
    // 64-element boxes, 128-byte swizzle. Null: the decode kernel stages with cp.async.
    const void* tmap = nullptr;
    const void* tmap64 = nullptr;  // the same view with 64-row boxes (prompt K/V tiles)
    const void* tmap_q = nullptr;  // the step's q buffer [max_rows][n_h][d_head] as (dims, heads,
                                   // rows) with 64 x G x 128/G boxes (tcgen05 prompt kernel)
};
// 2-D bf16 tensor map (rows x cols, K-major) with box_rows x box_cols boxes, 128-byte swizzle.
int make_tmap_2d_bf16(void* tmap_out, const void* base, uint64_t rows, uint64_t cols,
                      uint32_t box_rows, uint32_t box_cols);
// 3-D bf16 tensor map over [d2][d1][d0] (d0 contiguous), boxes b0 x b1 x b2, 128-byte swizzle.
int make_tmap_3d_bf16(void* tmap_out, const void* base, uint64_t d0, uint64_t d1, uint64_t d2,
                      uint32_t b0, uint32_t b1, uint32_t b2);

// Rotary embedding on q and k (rotate-half, table [max_pos][d_head/2] cos / sin) and
// the paged KV append of k, v for every row at row_pos[t] into page row_page[t].
// With planes, the qkv values are bf16(sum of planes) (the deferred GEMM epilogue).
void rope_kv_append(const __nv_bfloat16* qkv, int T, int n_h, int n_kv, int d_head,
                    const int32_t* row_pos, const int32_t* row_page, const float* rope_cos,
                    const float* rope_sin, const KvLayout& kv, int layer, __nv_bfloat16* q_out,
                    cudaStream_t stream, const Planes& planes = Planes{});

// Paged causal attention: row t attends positions [0, row_pos[t]] of its request, whose pages
// are flat_pages[row_page_off[t] ...]. Output o[T, n_h * d_head] bf16.
// Prompt query blocks: blocks[3*i] = first row, [3*i+1] = consecutive positions
// (<= attention_block_positions() rows of one request), [3*i+2] = 0. Decode rows (one query
// position each) are listed separately in drows[] and go to the decode kernel.
// Context splits: s_prompt for the prompt blocks, s_decode for the decode rows; each kernel's
// last CTA of a (row or block, KV head) merges the split partials (`counters`: zeroed ints,
// >= 2 x rows x n_kv, self-resetting; ws: rows x n_h x max(splits) x (d_head + 2) floats).
int attention_block_positions(int n_h, int n_kv, int d_head);
void attention_splits(int T, int n_h, int d_head, int n_blocks, int n_drows, int n_kv, int max_ctx,
                      int max_prompt_ctx, size_t ws_floats, int* s_prompt, int* s_decode);
int attention_launches(int n_blocks, int n_drows, int s_prompt, int s_decode);
size_t attention_workspace_floats(int T, int n_h, int d_head, int splits);
int attention_paged(const __nv_bfloat16* q, int T, int n_h, const int32_t* row_pos,
                    const int32_t* row_page_off, const int32_t* flat_pages, const int32_t* blocks,
                    int n_blocks, const int32_t* drows, int n_drows,
                    const KvLayout& kv, int layer, int s_prompt, int s_decode, __nv_bfloat16* o,
                    float* ws, size_t ws_floats, int* counters, const L2Prefetch& pf,
                    cudaStream_t stream);

// ids[r] = argmax_v logits[r, v] (lowest index wins ties).
void argmax_rows(const float* logits, int R, int V, int32_t* ids, cudaStream_t stream);
// last_token[req[r]] = ids[r]
void scatter_tokens(const int32_t* ids, const int32_t* req, int R, int32_t* last_token,
                    cudaStream_t stream);
// tokens[t] = prompt_tok[t] >= 0 ? prompt_tok[t] : last_token[row_req[t]]
void resolve_tokens(const int32_t* prompt_tok, const int32_t* row_req, const int32_t* last_token,
                    int T, int32_t* tokens, cudaStream_t stream);

// Eager module load of every kernel (see gemm_tc.cu preload_gemm).
void preload_gemm();
void preload_attention();
void preload_elementwise();
inline void preload_all() {
    preload_gemm();
    preload_attention();
    preload_elementwise();
}

}  // namespace ds
