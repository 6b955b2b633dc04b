/* TEST INFRASTRUCTURE ONLY — the CPU oracle of the stage forward. Never linked into the product.
 *
 * The reference (pipesim) has no arithmetic for the stage forward: it substitutes a calibration
 * lookup (src/perf_model.cpp:85-114, called at src/sim.cpp:424-425). This is the build's CPU
 * restatement of one Llama-3 pipeline stage under the conventions pinned in SURVEY.md Appendix C
 * (parity UNPINNED by the reference). */
#ifndef LLAMA_REF_H
#define LLAMA_REF_H
#include <stdint.h>

typedef struct lr_model {
    int32_t n_layers, d_model, n_heads, n_kv_heads, d_head, ffn, vocab, max_seq_len;
    float rope_theta, norm_eps;
} lr_model;

/* identical layout to ds_row (include/deserve.h) */
typedef struct lr_row {
    int32_t slot, pos, n_tok, need_logits, is_decode, reserved;
    int64_t req_id;
} lr_row;

typedef struct lr_stage lr_stage;

float lr_weight(uint64_t seed, uint64_t tensor_id, int64_t index, float scale);
int32_t lr_prompt_token(int64_t req_id, int32_t pos);
/* out[i] = lr_weight(seed, tensor_id, i, scale) for i < n (bf16 values held in fp32) */
void lr_fill_weights(uint64_t seed, uint64_t tensor_id, int64_t n, float scale, float* out);
lr_stage* lr_stage_create(const lr_model* m, int32_t layer_begin, int32_t layer_end,
                          int32_t is_first, int32_t is_last, uint64_t seed, int32_t max_handles);
void lr_stage_destroy(lr_stage* s);
/* forget every request's KV (timing harness: bounded memory between sampled circuits) */
void lr_stage_reset_kv(lr_stage* s);
/* tokens: first stage, one id per row position (T); act_in: other stages, [T, d] (bf16 values
 * held in fp32). act_out: [T, d]; logits: [R, vocab] fp32 (may be NULL); ids: [R]. */
int lr_stage_step(lr_stage* s, int32_t mb, int32_t max_slots, const lr_row* rows, int32_t n_rows,
                  const int32_t* tokens, const float* act_in, float* act_out, float* logits,
                  int32_t* ids);
#endif
