/*
 * deserve.h — C ABI of the B200-native DeServe stage-step path (libdeserve_b200.so).
 *
 * The reference (/root/reference/proj, "pipesim") has no GPU path: its stage forward is the
 * calibration lookup `scaled_stage_time()` (src/perf_model.cpp:109-114) called from
 * `Engine::on_compute_start` (src/sim.cpp:409-428); its swap is byte/time arithmetic in
 * `Engine::issue_swap_in` (src/sim.cpp:328-353); its hop is `Engine::send_onward`
 * (src/sim.cpp:430-439). Each entry point below is the call a maintainer binds at one of those
 * slots. Conventions: every call returns ds_status (0 = ok) and never throws or aborts;
 * ds_last_error() returns a thread-local message for the last failure. No torch types cross
 * this boundary: plain pointers, sizes and integers only.
 */
#ifndef DESERVE_B200_H
#define DESERVE_B200_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef int32_t ds_status;
#define DS_OK 0
#define DS_ERR_ARG 1        /* bad argument (maps to pipesim::ConfigError)               */
#define DS_ERR_PLAN 2       /* infeasible plan / device OOM (maps to pipesim::PlanError)  */
#define DS_ERR_RUNTIME 3    /* CUDA / NCCL / executor failure (maps to pipesim::SimError) */
#define DS_ERR_NO_DEVICE 4  /* no CUDA device visible: the product has no CPU fallback    */

const char* ds_last_error(void);
const char* ds_version(void);

/* ------------------------------------------------------------------------------------------
 * Integer hot path (bit-exact with the reference).
 * ------------------------------------------------------------------------------------------ */

/* Reference: stage_compute_time / scaled_stage_time (src/perf_model.cpp:85-114).
 * batch_sizes/times_us: the calibration table (batch strictly increasing). */
ds_status ds_stage_time_us(const int64_t* batch_sizes, const int64_t* times_us, int64_t n,
                           int64_t batch, int64_t layers, int64_t ref_layers, int64_t* out_us);

/* Reference: page_bytes / kv_bytes / global_pool_size (src/perf_model.cpp:116-136). */
ds_status ds_page_bytes(int64_t kv_bytes_per_token, int64_t layers, int64_t total_layers,
                        int64_t* out);
ds_status ds_global_pool_size(int64_t pcie_bw, int64_t stage_time_us, int64_t page,
                              int64_t* out);

/* Reference: memory_budget (src/perf_model.cpp:138-167). out5 = {M_KV, M_G, M_B, M_B', local}. */
ds_status ds_memory_budget(int64_t mem, int64_t weights, int64_t n_mb, int64_t m_global,
                           int32_t offload, int64_t* out5);
/* Reference: RequestGenerator::make (src/workload.cpp:36-53). out2 = {prompt_len, output_len}. */
ds_status ds_request_lengths(uint64_t seed, int64_t prompt_min, int64_t prompt_max, int64_t output_min,
                             int64_t output_max, int64_t index, int64_t* out2);
/* Reference: steady_state_throughput (src/sim.cpp:597-604) on a plan document. */
ds_status ds_steady_state_throughput(const char* plan_json, double* out);

/* Reference: plan() (src/planner.cpp:140-276) on a config document in the reference JSON format
 * (src/config.cpp:103-252). policy: NULL/"" = config as written, else "baseline" | "offload" |
 * "opt" (src/sweep.cpp:26-43). latency_us >= 0 overrides every link latency (sweep.cpp:45-49);
 * nb_override >= 0 overrides scheduler.nb_override. Writes the plan JSON (byte-identical to
 * PipelinePlan::to_json, src/planner.cpp:294-335) into out (NUL-terminated, truncated to cap);
 * *needed receives the full length. */
ds_status ds_plan_config(const char* config_json, const char* config_dir, const char* policy,
                         int64_t latency_us, int64_t nb_override, char* out, size_t cap,
                         size_t* needed);

/* Reference: run() (src/sim.cpp:591-595) in virtual-clock mode. The executor's own scheduler
 * (not the reference engine) produces the trace; write_trace format (src/trace.cpp:40-46).
 * trace_path may be NULL. report_json receives the SimReport fields (src/sim.cpp:501-532). */
ds_status ds_sim_config(const char* config_json, const char* config_dir, const char* policy,
                        int64_t latency_us, int64_t nb_override, const char* trace_path,
                        char* report_json, size_t cap);

/* Same, on an explicit plan document (PipelinePlan::from_json, src/planner.cpp:337-378) instead
 * of running the planner; the config supplies model, topology and workload. */
ds_status ds_sim_plan(const char* config_json, const char* config_dir, const char* plan_json,
                      const char* trace_path, char* report_json, size_t cap);

/* The recorded schedule the GPU executor replays: {"circuits": [{mb, eff_batch, n_decode, t_end,
 * rows: [[slot,pos,n_tok,need_logits,is_decode,req_id]...], completed: [slot...]}...],
 * "ops": per stage [[kind(0 compute,1 swap-in,2 release), mb, slot, circuit, plan_bytes, t_us]...]}. */
ds_status ds_schedule_config(const char* config_json, const char* config_dir, const char* policy,
                             int64_t latency_us, int64_t nb_override, int64_t max_circuits, char* out,
                             size_t cap, size_t* needed);

/* ------------------------------------------------------------------------------------------
 * Stage forward (the compute slot of Engine::on_compute_start, src/sim.cpp:424-425).
 * ------------------------------------------------------------------------------------------ */

typedef struct ds_model_desc {
    int32_t n_layers;      /* whole model */
    int32_t d_model;
    int32_t n_heads;
    int32_t n_kv_heads;
    int32_t d_head;
    int32_t ffn;
    int32_t vocab;
    int32_t max_seq_len;
    float rope_theta;      /* 500000 for Llama 3 */
    float norm_eps;        /* 1e-5 */
} ds_model_desc;

/* One row group of a circuit: n_tok consecutive positions [pos, pos+n_tok) of the request in
 * microbatch slot `slot`. Decode rows have n_tok == 1; prefill rows carry up to prefill_chunk
 * prompt positions (reference begin_circuit, src/sim.cpp:386-407). need_logits = 1 samples a
 * token from the group's last position (decode rows, and the prefill group completing a prompt). */
typedef struct ds_row {
    int32_t slot;
    int32_t pos;
    int32_t n_tok;
    int32_t need_logits;
    int32_t is_decode;     /* 1: decode row (input = token sampled last circuit); 0: prompt rows */
    int32_t reserved;
    int64_t req_id;
} ds_row;

/* Synthetic prompt token of request req_id at position pos (BOS = 128000 at position 0;
 * otherwise SplitMix64(0x5EED ^ req_id * phi ^ pos) mod 128000). The reference has no token ids
 * (SURVEY.md Appendix C); this is the build's pinned convention, shared with the CPU oracle. */
int32_t ds_prompt_token_id(int64_t req_id, int32_t pos);

typedef struct ds_stage ds_stage;

ds_status ds_stage_create(int32_t device, const ds_model_desc* model, int64_t layer_begin,
                          int64_t layer_end, int32_t is_first, int32_t is_last,
                          uint64_t weight_seed, int32_t max_rows, int32_t max_slots,
                          ds_stage** out);
ds_status ds_stage_destroy(ds_stage* stage);

/* KV pool of the stage (reference MemoryBudget, include/pipesim/perf_model.hpp:57-72 and the swap
 * plan of src/sim.cpp:296-353). page_bytes must equal reference page_bytes(). Device pages:
 * n_mb * floor(local_bytes_per_mb / page) local + 2 * global_slot_bytes / page slot pages;
 * pinned host backing of host_bytes_per_mb per microbatch. */
ds_status ds_kv_create(ds_stage* stage, int64_t page_bytes, int64_t n_mb, int64_t local_bytes_per_mb,
                       int64_t global_slot_bytes, int64_t host_bytes_per_mb);
/* The request in (mb, slot) completed: free its pages (reference on_compute_end, sim.cpp:462-468). */
ds_status ds_kv_release(ds_stage* stage, int32_t mb, int32_t slot);
/* Bytes of KV pages the microbatch holds / holds outside its local pool. */
ds_status ds_kv_usage(ds_stage* stage, int32_t mb, int64_t* total_bytes, int64_t* global_bytes);

/* Frees every page of every microbatch (pools and pinned backing stay allocated). */
ds_status ds_kv_reset(ds_stage* stage);
/* Enables CUDA-event timing around every launch group of ds_stage_step (clears the records). */
ds_status ds_stage_profile(ds_stage* stage, int32_t enable);
/* JSON {kind: {n, ms, flops, bytes, rows}} for kinds gemm_qkv, attention, gemm_o, gemm_gate_up,
 * gemm_down, gemm_lm_head, elementwise (algorithmic FLOPs / bytes); *launches = kernel
 * launches issued by this stage since creation. Clears the timing records. */
ds_status ds_stage_kernel_stats(ds_stage* stage, char* out, size_t cap, int64_t* launches);
/* 1 if every KV page of mb is device-resident (compute-requires-resident, sim.cpp:629-639). */
ds_status ds_kv_resident(ds_stage* stage, int32_t mb, int32_t* resident);
/* 1 if mb is resident AND the pages this step's rows append fit its free local pages (plus its
 * global slot's free pages when it holds one); 0 means the caller must swap mb in first -- the
 * on-demand swap-in of reference try_start (sim.cpp:355-382) for growth the plan's byte-level
 * prefetch did not cover (local capacity is whole pages). */
ds_status ds_kv_ready(ds_stage* stage, int32_t mb, const ds_row* rows, int64_t n_rows, int32_t* ready);

/* H2D prefetch of mb's global pages into global slot `slot` after evicting the occupant (D2H),
 * on the stage's copy streams (reference issue_swap_in, sim.cpp:328-353). plan_bytes is the
 * reference's integer contract (logged); the copy moves whole pages. The refill of a slot page
 * waits only for that page's eviction, so both directions run at once; the microbatch's next
 * ds_stage_step waits for both. moved_in/out may be NULL. */
ds_status ds_swap_in(ds_stage* stage, int32_t mb, int32_t slot, int64_t plan_bytes,
                     int64_t* moved_in, int64_t* moved_out);

/* Bytes of the last ds_swap_in: out4 = {refill into the global slot (compare with plan_bytes;
 * <= plan + 1 page), migration into local pages freed by completions, eviction, page copies}.
 * Copies move only the occupied tokens of a partial page (one 2D copy per page). */
ds_status ds_swap_stats(ds_stage* stage, int64_t* out4);

/* One stage step of microbatch mb over `rows`. act_in: first stage = device int32 ids sampled by
 * the previous circuit of this mb (NULL on its first circuit); other stages = device bf16
 * [T, d_model]. act_out: last stage = device int32 ids [R] (R = rows with need_logits); other
 * stages = device bf16 [T, d_model]. NULL act_out keeps the result in the stage buffer
 * (ds_stage_output). The step is stream-ordered; ds_stage_sync waits for it. */
ds_status ds_stage_step(ds_stage* stage, int32_t mb, const ds_row* rows, int64_t n_rows,
                        const void* act_in, void* act_out);
ds_status ds_stage_output(ds_stage* stage, void** ptr, int64_t* bytes, int64_t* n_out);
ds_status ds_stage_sync(ds_stage* stage);
ds_status ds_stage_stream(ds_stage* stage, void** cuda_stream);
/* Real-clock trace hooks (the executor's EventTrace, reference trace.hpp:24-42). The events
 * (cudaEvent_t, created by the caller) are recorded once, by the NEXT call only:
 * ds_stage_step: ready = the step reached the stream (before its swap-in wait), start = after
 * that wait (ComputeStart), end = after its last kernel (ComputeEnd);
 * ds_swap_in: in0/in1 bracket the H2D refill, out0/out1 the D2H eviction (Swap{In,Out}Done).
 * Any event may be NULL. */
ds_status ds_stage_step_events(ds_stage* stage, void* ready, void* start, void* end);
ds_status ds_swap_events(ds_stage* stage, void* in0, void* in1, void* out0, void* out1);
/* Device pointer to the fp32 logits [rows x vocab] of the last step (valid until the next step;
 * stream-ordered on ds_stage_stream). */
ds_status ds_stage_logits_device(ds_stage* stage, const float** ptr, int64_t* rows);
/* Teacher forcing / debugging: read the fp32 logits of the last step (R x vocab) to host. */
ds_status ds_stage_logits(ds_stage* stage, float* host_out, int64_t max_floats, int64_t* n_floats);

/* ------------------------------------------------------------------------------------------
 * Whole-pipeline GPU run (the reference's run() with real stage forwards; replay mode).
 * ------------------------------------------------------------------------------------------ */
typedef struct ds_gpu_opts {
    int32_t device0;        /* first CUDA device */
    int32_t n_devices;      /* 0 = all visible; stage s runs on device0 + s % n_devices */
    int32_t real_delay;     /* 1: a hop may not arrive before completion + latency + bytes/bw */
    int32_t collect_tokens; /* 1: report the sampled ids of every circuit */
    int64_t max_circuits;   /* execute the first circuits of the schedule (0 = all) */
    uint64_t weight_seed;
    int32_t trace;          /* 1: keep the schedule's events; ds_session_trace rebuilds them on
                               the real clock after every run */
    int32_t reserved;
} ds_gpu_opts;

/* Plans the config (as ds_plan_config), schedules it in virtual time, then executes the schedule on
 * GPUs: per stage, computes / swap-ins / releases in schedule order, hops with injected delay.
 * report_json: circuits, decode tokens, wall time, per-stage busy time and (rows, ms) per step,
 * swap plan vs moved bytes, residency top-ups, optionally the sampled ids. */
ds_status ds_gpu_run_config(const char* config_json, const char* config_dir, const char* policy,
                            int64_t latency_us, int64_t nb_override, const ds_model_desc* model,
                            const ds_gpu_opts* opts, char* report_json, size_t cap, size_t* needed);

/* The same run as a reusable session: stages and weights are created once; every ds_session_run
 * replays the schedule from empty KV pools (bench warm-up / timed runs). profile = 1 adds CUDA
 * events around every launch group (report "kernels": algorithmic FLOPs/bytes and ms per kind). */
typedef struct ds_session ds_session;
ds_status ds_session_create(const char* config_json, const char* config_dir, const char* policy,
                            int64_t latency_us, int64_t nb_override, const ds_model_desc* model,
                            const ds_gpu_opts* opts, ds_session** out);
ds_status ds_session_run(ds_session* session, int32_t profile, int32_t collect_tokens,
                         char* report_json, size_t cap, size_t* needed);
ds_status ds_session_destroy(ds_session* session);

/* Reference SimResult{report, trace} of a hardware run (include/pipesim/sim.hpp:47-51): the
 * events of the last ds_session_run on the real clock, in write_trace format
 * (src/trace.cpp:40-46), integer fields identical to the virtual-clock schedule's (replay mode;
 * GPU event times mapped to the host steady clock, hop arrivals from the host), so reference
 * replay_check (sim.cpp:606-697) and windowed_stats (workload.cpp:82-116) accept it unchanged.
 * Needs opts.trace = 1. trace_path may be NULL. t0_us: steady-clock origin in us (< 0: this
 * run's start; ranks of one pipeline pass a common origin). keep_virtual_seq = 1 writes the
 * schedule's seq numbers (for ds_trace_merge of per-rank traces), else seq = line index.
 * report_json: SimReport fields (build_report, sim.cpp:501-532) over [w0_us, w1_us) of this
 * process's events (w0 < 0: workload warmup; w1 < 0: min(bench duration, run end)), plus
 * "replay": the executed circuits/events. */
ds_status ds_session_trace(ds_session* session, const char* trace_path, int64_t t0_us,
                           int32_t keep_virtual_seq, int64_t w0_us, int64_t w1_us, char* report_json,
                           size_t cap, size_t* needed);
/* Later runs execute only the first max_circuits circuits of the prefix prepared at creation
 * (0 = all of it: warm-up runs on a short prefix, then the measured run). *t0_us (may be NULL)
 * receives the host steady-clock start of the last run (ranks agree on a common trace origin). */
ds_status ds_session_limit(ds_session* session, int64_t max_circuits, int64_t* t0_us);
/* Merges per-rank traces (each sorted, virtual seq kept) into one trace in (time, seq) order with
 * seq renumbered as the line index. */
ds_status ds_trace_merge(const char* const* paths, int32_t n_paths, const char* out_path);
/* SimReport fields of a trace file over [w0_us, w1_us) (windowed_stats token counts; busy /
 * swap-stall / bubble per stage as the engine accumulates them). */
ds_status ds_trace_report(const char* trace_path, int64_t n_stages, int64_t w0_us, int64_t w1_us,
                          uint64_t seed, char* report_json, size_t cap);
/* The reference's report.kv (report_to_kv, src/sweep.cpp:146-195; no pricing block) of a report
 * JSON (ds_run / ds_session_trace / ds_sim_config "report") on its plan document. */
ds_status ds_report_kv(const char* report_json, const char* plan_json, int64_t latency_us,
                       const char* policy, char* out, size_t cap, size_t* needed);
/* report_kv with the pricing block (report_to_kv with a ProfitAnalysis, src/sweep.cpp:187-194):
 * pricing_json is a config document's "pricing" object ({"preset": name} or the money fields,
 * src/config.cpp:169-199); the analysis is the reference's analyze (src/economics.cpp:21-59).
 * DS_ERR_ARG on a bad pricing object or a zero unified price, DS_ERR_RUNTIME on an empty window. */
ds_status ds_report_kv_priced(const char* report_json, const char* plan_json, int64_t latency_us,
                              const char* policy, const char* pricing_json, char* out, size_t cap,
                              size_t* needed);
/* The reference's sweep.csv (SweepResult::to_csv, src/sweep.cpp:68-82): policies x latencies
 * output throughputs (row-major; NaN = failed cell). policies: comma-separated names. */
ds_status ds_sweep_csv(const int64_t* latencies_us, int32_t n_latencies, const char* policies,
                       const double* throughput, char* out, size_t cap, size_t* needed);
/* The drop-in execution seam: the reference's run(plan, topo, workload, model)
 * (src/sim.cpp:591-595) with real stage forwards. Plans the config (ds_plan_config), schedules it,
 * executes it on GPUs, writes the real-clock trace to trace_path (may be NULL) and returns
 * {"report": SimReport over the workload window clipped to the run, "gpu": the executor report}. */
ds_status ds_run(const char* config_json, const char* config_dir, const char* policy,
                 int64_t latency_us, int64_t nb_override, const ds_model_desc* model,
                 const ds_gpu_opts* opts, const char* trace_path, char* report_json, size_t cap,
                 size_t* needed);
/* Teacher-forced parity (tests): every run copies the fp32 logits of the rows sampled for these
 * requests to host memory; ds_session_captured returns them in execution order with meta
 * [circuit, req_id, position, row within the circuit's sampled rows] per row. */
ds_status ds_session_capture(ds_session* session, const int64_t* req_ids, int64_t n);
ds_status ds_session_captured(ds_session* session, int64_t* meta4, float* logits, int64_t max_rows,
                              int64_t* n_rows);

/* One process per GPU: this process runs pipeline stage `rank` of `world` (= stages) on device0;
 * activations (and sampled ids, last -> first) hop over NCCL send/recv, one 2-rank communicator per
 * ring link (reference ring links, src/planner.cpp:122-138). nccl_ids: world x 128 bytes, id i for
 * link i -> i+1, generated once (ds_nccl_unique_id) and shared by the launcher. */
ds_status ds_nccl_unique_id(uint8_t* out128);
ds_status ds_session_create_rank(const char* config_json, const char* config_dir, const char* policy,
                                 int64_t latency_us, int64_t nb_override, const ds_model_desc* model,
                                 const ds_gpu_opts* opts, int32_t rank, int32_t world,
                                 const uint8_t* nccl_ids, ds_session** out);

/* ------------------------------------------------------------------------------------------
 * Kernel-level entry points (parity tests call these through the same library).
 * ------------------------------------------------------------------------------------------ */
ds_status ds_dbg_gemm(const uint16_t* x, const uint16_t* w, int32_t T, int32_t N, int32_t K,
                      int32_t epi, const uint16_t* resid, int32_t k_splits, void* out);
/* RowNorm pair: out_x = bf16(resid + bf16(x.W1^T)) [T, N] (producer, slice sums of squares in
 * its epilogue), then out_y = bf16(r[t] * out_x[t].W2^T) [T, N2], r = 1/sqrt(mean(out_x^2) + eps)
 * (consumer row scale; *fused = 1) — or, where a partition does not allow it (*fused = 0), the
 * RMSNorm kernel and the plain GEMM of bf16(out_x * r). */
ds_status ds_dbg_gemm_norm(const uint16_t* x, const uint16_t* w1, int32_t T, int32_t N, int32_t K,
                           const uint16_t* resid, const uint16_t* w2, int32_t N2, float eps,
                           uint16_t* out_x, uint16_t* out_y, int32_t* fused);
ds_status ds_dbg_gemm_bench(int32_t T, int32_t N, int32_t K, int32_t epi, int32_t iters,
                            int32_t k_splits, float* ms_out);
/* The GEMM work partition for a [T x K] . [N x K]^T product, host arithmetic only (no device):
 * out[12] = {0, CTAs per cluster, clusters, data-parallel rounds, stream-K remainder tiles,
 * stream-K clusters, k-split ways, planes, deferred finish, tokens per block, token blocks,
 * k-blocks per tile}. */
ds_status ds_dbg_gemm_plan(int32_t T, int32_t N, int32_t K, int32_t* out);
ds_status ds_dbg_has_device(int32_t* n_devices);
ds_status ds_dbg_alloc(int32_t device, int64_t bytes, void** out);
ds_status ds_dbg_free(void* ptr);
/* synchronous copy in any direction (cudaMemcpyDefault, unified addressing) */
ds_status ds_dbg_copy(void* dst, const void* src, int64_t bytes);

#ifdef __cplusplus
}
#endif
#endif /* DESERVE_B200_H */
