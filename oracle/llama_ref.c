/* TEST INFRASTRUCTURE ONLY — CPU oracle of one Llama-3 pipeline stage (see llama_ref.h).
 *
 * Numerics (the contract the sm_100a kernels follow):
 *   storage bf16 (held here as bf16-rounded fp32), fp32 accumulation;
 *   RMSNorm  y = bf16(g * bf16(x * 1/sqrtf(mean(x^2) + eps)))            (HF LlamaRMSNorm order)
 *   QKV      bf16(x . W^T), RoPE rotate-half theta=500000 on q,k, table cos/sin(pos*theta^(-2i/dh))
 *            evaluated in double and stored fp32; out = bf16(x1*c - x2*s), bf16(x2*c + x1*s)
 *   attn     causal over positions [0, pos], GQA head h -> kv head h/(n_h/n_kv), fp32 softmax
 *   O, down  x = bf16(x + bf16(acc))   (residual add after rounding the projection)
 *   MLP      h = bf16(bf16(silu(bf16(g))) * bf16(u)), silu(v) = v / (1 + expf(-v))
 *   head     final RMSNorm on the sampled rows, fp32 logits, argmax lowest index on ties
 * Weights: w = bf16((2u - 1) * scale), u = (mix64(seed + id*phi + i*C) >> 40) / 2^24, the same
 * counter hash the GPU init kernel uses; scale = sqrt(3 / fan_in) (embedding 1.0), norms = 1.
 */
#include "llama_ref.h"

#include <math.h>
#include <stdlib.h>
#include <string.h>

static uint64_t mix64(uint64_t z) {
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ULL;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBULL;
    return z ^ (z >> 31);
}

static float bf(float x) { /* round to bf16, RNE */
    uint32_t u;
    memcpy(&u, &x, 4);
    u = (u + 0x7FFFu + ((u >> 16) & 1u)) & 0xFFFF0000u;
    float r;
    memcpy(&r, &u, 4);
    return r;
}

static uint16_t bf_bits(float x) {
    uint32_t u;
    memcpy(&u, &x, 4);
    return (uint16_t)((u + 0x7FFFu + ((u >> 16) & 1u)) >> 16);
}

static float from_bits(uint16_t b) {
    uint32_t u = (uint32_t)b << 16;
    float r;
    memcpy(&r, &u, 4);
    return r;
}

float lr_weight(uint64_t seed, uint64_t tensor_id, int64_t index, float scale) {
    const uint64_t h = mix64(seed + tensor_id * 0x9E3779B97F4A7C15ULL + (uint64_t)index * 0xD1B54A32D192ED03ULL);
    const float u = (float)(h >> 40) * (1.0f / 16777216.0f);
    return bf((2.0f * u - 1.0f) * scale);
}

void lr_fill_weights(uint64_t seed, uint64_t tensor_id, int64_t n, float scale, float* out) {
#pragma omp parallel for schedule(static)
    for (int64_t i = 0; i < n; ++i) out[i] = lr_weight(seed, tensor_id, i, scale);
}

int32_t lr_prompt_token(int64_t req_id, int32_t pos) {
    if (pos == 0) return 128000;
    uint64_t z = 0x5EEDULL ^ ((uint64_t)req_id * 0x9E3779B97F4A7C15ULL) ^ (uint64_t)pos;
    z += 0x9E3779B97F4A7C15ULL;
    z = mix64(z);
    return (int32_t)(z % 128000ULL);
}

typedef struct {
    uint16_t *wq, *wk, *wv, *wo, *wg, *wu, *wd; /* canonical [out][in] bf16 bits */
} layer_w;

typedef struct {
    int64_t req_id;
    int cap;      /* positions held per (layer, K|V, kv head); grows on demand */
    uint16_t* kv; /* [L][2][n_kv][cap][dh] bf16 bits (K after RoPE and V are bf16 values) */
} handle_kv;

/* make room for positions [0, need) keeping the cached ones; new positions are zero */
static void kv_reserve(handle_kv* hk, int L, int nkv, int dh, int need) {
    if (need <= hk->cap) return;
    int cap = hk->cap ? hk->cap : 256;
    while (cap < need) cap *= 2;
    uint16_t* nk = (uint16_t*)calloc((size_t)L * 2 * nkv * cap * dh, sizeof(uint16_t));
    if (hk->kv)
        for (size_t blk = 0; blk < (size_t)L * 2 * nkv; ++blk)
            memcpy(nk + blk * cap * dh, hk->kv + blk * hk->cap * dh, sizeof(uint16_t) * (size_t)hk->cap * dh);
    free(hk->kv);
    hk->kv = nk;
    hk->cap = cap;
}

struct lr_stage {
    lr_model m;
    int lb, le, L, first, last;
    uint64_t seed;
    layer_w* lw;
    uint16_t* lm; /* [vocab][d] */
    float *rc, *rs;
    int max_handles;
    handle_kv* h;
};

static uint16_t* gen(uint64_t seed, uint64_t id, int64_t rows, int64_t cols, float scale) {
    uint16_t* w = (uint16_t*)malloc(sizeof(uint16_t) * rows * cols);
#pragma omp parallel for schedule(static)
    for (int64_t i = 0; i < rows * cols; ++i) w[i] = bf_bits(lr_weight(seed, id, i, scale));
    return w;
}

lr_stage* lr_stage_create(const lr_model* m, int32_t lb, int32_t le, int32_t first, int32_t last,
                          uint64_t seed, int32_t max_handles) {
    lr_stage* s = (lr_stage*)calloc(1, sizeof(lr_stage));
    s->m = *m;
    s->lb = lb;
    s->le = le;
    s->L = le - lb;
    s->first = first;
    s->last = last;
    s->seed = seed;
    const int d = m->d_model, qd = m->n_heads * m->d_head, kvd = m->n_kv_heads * m->d_head;
    const float sd = (float)sqrt(3.0 / d), sq = (float)sqrt(3.0 / qd), sf = (float)sqrt(3.0 / m->ffn);
    s->lw = (layer_w*)calloc(s->L, sizeof(layer_w));
    for (int i = 0; i < s->L; ++i) {
        const uint64_t base = (uint64_t)(lb + i) * 16;
        s->lw[i].wq = gen(seed, base + 1, qd, d, sd);
        s->lw[i].wk = gen(seed, base + 2, kvd, d, sd);
        s->lw[i].wv = gen(seed, base + 3, kvd, d, sd);
        s->lw[i].wo = gen(seed, base + 4, d, qd, sq);
        s->lw[i].wg = gen(seed, base + 6, m->ffn, d, sd);
        s->lw[i].wu = gen(seed, base + 7, m->ffn, d, sd);
        s->lw[i].wd = gen(seed, base + 8, d, m->ffn, sf);
    }
    if (last) s->lm = gen(seed, (1ULL << 20) + 1, m->vocab, d, sd);
    const int half = m->d_head / 2;
    s->rc = (float*)malloc(sizeof(float) * (size_t)m->max_seq_len * half);
    s->rs = (float*)malloc(sizeof(float) * (size_t)m->max_seq_len * half);
    for (int p = 0; p < m->max_seq_len; ++p)
        for (int i = 0; i < half; ++i) {
            const double inv = pow((double)m->rope_theta, -2.0 * i / m->d_head);
            const double a = (double)p * inv;
            s->rc[(size_t)p * half + i] = (float)cos(a);
            s->rs[(size_t)p * half + i] = (float)sin(a);
        }
    s->max_handles = max_handles;
    s->h = (handle_kv*)calloc(max_handles, sizeof(handle_kv));
    for (int i = 0; i < max_handles; ++i) s->h[i].req_id = -1;
    return s;
}

void lr_stage_reset_kv(lr_stage* s) {
    for (int i = 0; i < s->max_handles; ++i) {
        free(s->h[i].kv);
        s->h[i].kv = NULL;
        s->h[i].cap = 0;
        s->h[i].req_id = -1;
    }
}

void lr_stage_destroy(lr_stage* s) {
    if (!s) return;
    for (int i = 0; i < s->L; ++i) {
        free(s->lw[i].wq); free(s->lw[i].wk); free(s->lw[i].wv); free(s->lw[i].wo);
        free(s->lw[i].wg); free(s->lw[i].wu); free(s->lw[i].wd);
    }
    free(s->lw);
    free(s->lm);
    free(s->rc);
    free(s->rs);
    for (int i = 0; i < s->max_handles; ++i) free(s->h[i].kv);
    free(s->h);
    free(s);
}

/* y[t][n] = sum_k x[t][k] * w[n][k], fp32: per (t, n) 16 partial sums (lane j takes k = j mod 16)
 * then a fixed-order reduction. Rows are processed 4 at a time against one converted weight row
 * (the per-(t, n) summation order is unchanged, so results do not depend on the blocking). */
static float dot1(const float* x, int K, const float* wf) {
    float acc[16] = {0};
    int k = 0;
    for (; k + 16 <= K; k += 16)
        for (int j = 0; j < 16; ++j) acc[j] += x[k + j] * wf[k + j];
    float sum = 0.f;
    for (int j = 0; j < 16; ++j) sum += acc[j];
    for (; k < K; ++k) sum += x[k] * wf[k];
    return sum;
}

static void dot4(const float* x, int K, const float* wf, float* out) {
    const float *x0 = x, *x1 = x + K, *x2 = x + 2 * (size_t)K, *x3 = x + 3 * (size_t)K;
    float a0[16] = {0}, a1[16] = {0}, a2[16] = {0}, a3[16] = {0};
    int k = 0;
    for (; k + 16 <= K; k += 16)
        for (int j = 0; j < 16; ++j) {
            const float wv = wf[k + j];
            a0[j] += x0[k + j] * wv;
            a1[j] += x1[k + j] * wv;
            a2[j] += x2[k + j] * wv;
            a3[j] += x3[k + j] * wv;
        }
    float* acc[4] = {a0, a1, a2, a3};
    const float* xs[4] = {x0, x1, x2, x3};
    for (int r = 0; r < 4; ++r) {
        float sum = 0.f;
        for (int j = 0; j < 16; ++j) sum += acc[r][j];
        for (int kk = k; kk < K; ++kk) sum += xs[r][kk] * wf[kk];
        out[r] = sum;
    }
}

static void matmul(const float* x, int T, int K, const uint16_t* w, int N, float* y) {
    enum { NBLK = 8 }; /* weight rows converted at once: x blocks are reused across them */
    const int nblocks = (N + NBLK - 1) / NBLK;
#pragma omp parallel
    {
        float* wf = (float*)malloc(sizeof(float) * (size_t)K * NBLK);
#pragma omp for schedule(static)
        for (int b = 0; b < nblocks; ++b) {
            const int n0 = b * NBLK, nn = N - n0 < NBLK ? N - n0 : NBLK;
            for (int i = 0; i < nn; ++i) {
                const uint16_t* wr = w + (size_t)(n0 + i) * K;
                for (int k = 0; k < K; ++k) wf[(size_t)i * K + k] = from_bits(wr[k]);
            }
            int t = 0;
            for (; t + 4 <= T; t += 4)
                for (int i = 0; i < nn; ++i) {
                    float o[4];
                    dot4(x + (size_t)t * K, K, wf + (size_t)i * K, o);
                    for (int r = 0; r < 4; ++r) y[(size_t)(t + r) * N + n0 + i] = o[r];
                }
            for (; t < T; ++t)
                for (int i = 0; i < nn; ++i)
                    y[(size_t)t * N + n0 + i] = dot1(x + (size_t)t * K, K, wf + (size_t)i * K);
        }
        free(wf);
    }
}

static void rmsnorm(const float* x, int d, float eps, float* y) {
    float ss = 0.f;
    for (int i = 0; i < d; ++i) ss += x[i] * x[i];
    const float r = 1.0f / sqrtf(ss / (float)d + eps);
    for (int i = 0; i < d; ++i) y[i] = bf(1.0f * bf(x[i] * r)); /* gains are 1.0 */
}

int lr_stage_step(lr_stage* s, int32_t mb, int32_t max_slots, const lr_row* rows, int32_t n_rows,
                  const int32_t* tokens, const float* act_in, float* act_out, float* logits,
                  int32_t* ids) {
    const lr_model* m = &s->m;
    const int d = m->d_model, nh = m->n_heads, nkv = m->n_kv_heads, dh = m->d_head;
    const int qd = nh * dh, kvd = nkv * dh, G = nh / nkv, half = dh / 2;
    int T = 0, R = 0;
    for (int i = 0; i < n_rows; ++i) {
        T += rows[i].n_tok;
        R += rows[i].need_logits ? 1 : 0;
    }
    int* row_h = (int*)malloc(sizeof(int) * T);
    int* row_pos = (int*)malloc(sizeof(int) * T);
    int* lrow = (int*)malloc(sizeof(int) * (R + 1));
    {
        int t = 0, r = 0;
        for (int i = 0; i < n_rows; ++i) {
            const int hidx = mb * max_slots + rows[i].slot;
            if (hidx >= s->max_handles) return -1;
            handle_kv* hk = &s->h[hidx];
            if (hk->req_id != rows[i].req_id) hk->req_id = rows[i].req_id;
            kv_reserve(hk, s->L, nkv, dh, rows[i].pos + rows[i].n_tok);
            for (int j = 0; j < rows[i].n_tok; ++j, ++t) {
                row_h[t] = hidx;
                row_pos[t] = rows[i].pos + j;
            }
            if (rows[i].need_logits) lrow[r++] = t - 1;
        }
    }
    float* x = (float*)malloc(sizeof(float) * (size_t)T * d);
    float* xn = (float*)malloc(sizeof(float) * (size_t)T * d);
    float* q = (float*)malloc(sizeof(float) * (size_t)T * qd);
    float* kk = (float*)malloc(sizeof(float) * (size_t)T * kvd);
    float* vv = (float*)malloc(sizeof(float) * (size_t)T * kvd);
    float* att = (float*)malloc(sizeof(float) * (size_t)T * qd);
    float* acc = (float*)malloc(sizeof(float) * (size_t)T * (m->ffn > d ? m->ffn : d));
    float* g = (float*)malloc(sizeof(float) * (size_t)T * m->ffn);
    float* u = (float*)malloc(sizeof(float) * (size_t)T * m->ffn);

    if (s->first) {
        for (int t = 0; t < T; ++t)
            for (int i = 0; i < d; ++i)
                x[(size_t)t * d + i] = lr_weight(s->seed, 1ULL << 20, (int64_t)tokens[t] * d + i, 1.0f);
    } else {
        memcpy(x, act_in, sizeof(float) * (size_t)T * d);
    }

    for (int li = 0; li < s->L; ++li) {
        const layer_w* w = &s->lw[li];
        for (int t = 0; t < T; ++t) rmsnorm(x + (size_t)t * d, d, m->norm_eps, xn + (size_t)t * d);
        matmul(xn, T, d, w->wq, qd, q);
        matmul(xn, T, d, w->wk, kvd, kk);
        matmul(xn, T, d, w->wv, kvd, vv);
        for (int t = 0; t < T; ++t) {
            const int p = row_pos[t];
            const float* c = s->rc + (size_t)p * half;
            const float* sn = s->rs + (size_t)p * half;
            for (int hh = 0; hh < nh + nkv; ++hh) {
                float* v = hh < nh ? q + (size_t)t * qd + hh * dh : kk + (size_t)t * kvd + (hh - nh) * dh;
                for (int i = 0; i < dh; ++i) v[i] = bf(v[i]);
                for (int i = 0; i < half; ++i) {
                    const float x1 = v[i], x2 = v[i + half];
                    const float o1 = x1 * c[i] - x2 * sn[i];
                    const float o2 = x2 * c[i] + x1 * sn[i];
                    v[i] = bf(o1);
                    v[i + half] = bf(o2);
                }
            }
            const size_t S = (size_t)s->h[row_h[t]].cap;
            uint16_t* kvb = s->h[row_h[t]].kv + (size_t)li * 2 * kvd * S;
            for (int kh = 0; kh < nkv; ++kh)
                for (int i = 0; i < dh; ++i) {
                    kvb[((size_t)kh * S + p) * dh + i] = bf_bits(kk[(size_t)t * kvd + kh * dh + i]);
                    kvb[((size_t)(nkv + kh) * S + p) * dh + i] = bf_bits(vv[(size_t)t * kvd + kh * dh + i]);
                }
        }
        const float scale = 1.0f / sqrtf((float)dh);
#pragma omp parallel for collapse(2) schedule(dynamic)
        for (int t = 0; t < T; ++t)
            for (int hh = 0; hh < nh; ++hh) {
                const int p = row_pos[t], kh = hh / G;
                const size_t S = (size_t)s->h[row_h[t]].cap;
                const uint16_t* kvb = s->h[row_h[t]].kv + (size_t)li * 2 * kvd * S;
                const float* qv = q + (size_t)t * qd + hh * dh;
                float* sc = (float*)malloc(sizeof(float) * (p + 1));
                float mx = -INFINITY;
                for (int j = 0; j <= p; ++j) {
                    const uint16_t* kr = kvb + ((size_t)kh * S + j) * dh;
                    float dot = 0.f;
                    for (int i = 0; i < dh; ++i) dot += qv[i] * from_bits(kr[i]);
                    sc[j] = dot * scale;
                    if (sc[j] > mx) mx = sc[j];
                }
                float sum = 0.f;
                for (int j = 0; j <= p; ++j) {
                    sc[j] = expf(sc[j] - mx);
                    sum += sc[j];
                }
                float* o = att + (size_t)t * qd + hh * dh;
                for (int i = 0; i < dh; ++i) o[i] = 0.f;
                for (int j = 0; j <= p; ++j) {
                    const uint16_t* vr = kvb + ((size_t)(nkv + kh) * S + j) * dh;
                    for (int i = 0; i < dh; ++i) o[i] += sc[j] * from_bits(vr[i]);
                }
                for (int i = 0; i < dh; ++i) o[i] = bf(o[i] / sum);
                free(sc);
            }
        matmul(att, T, qd, w->wo, d, acc);
        for (size_t i = 0; i < (size_t)T * d; ++i) x[i] = bf(x[i] + bf(acc[i]));
        for (int t = 0; t < T; ++t) rmsnorm(x + (size_t)t * d, d, m->norm_eps, xn + (size_t)t * d);
        matmul(xn, T, d, w->wg, m->ffn, g);
        matmul(xn, T, d, w->wu, m->ffn, u);
        for (size_t i = 0; i < (size_t)T * m->ffn; ++i) {
            const float gb = bf(g[i]);
            const float sg = bf(gb / (1.0f + expf(-gb)));
            g[i] = bf(sg * bf(u[i]));
        }
        matmul(g, T, m->ffn, w->wd, d, acc);
        for (size_t i = 0; i < (size_t)T * d; ++i) x[i] = bf(x[i] + bf(acc[i]));
    }
    if (act_out) memcpy(act_out, x, sizeof(float) * (size_t)T * d);
    if (s->last && R > 0) {
        float* xr = (float*)malloc(sizeof(float) * (size_t)R * d);
        for (int r = 0; r < R; ++r) rmsnorm(x + (size_t)lrow[r] * d, d, m->norm_eps, xr + (size_t)r * d);
        float* lg = logits ? logits : (float*)malloc(sizeof(float) * (size_t)R * m->vocab);
        matmul(xr, R, d, s->lm, m->vocab, lg);
        for (int r = 0; r < R; ++r) {
            const float* row = lg + (size_t)r * m->vocab;
            int best = 0;
            for (int v = 1; v < m->vocab; ++v)
                if (row[v] > row[best]) best = v;
            if (ids) ids[r] = best;
        }
        if (!logits) free(lg);
        free(xr);
    }
    free(x); free(xn); free(q); free(kk); free(vv); free(att); free(acc); free(g); free(u);
    free(row_h); free(row_pos); free(lrow);
    return 0;
}
