// GPU replay executor (executor.cpp): drives ds_stage objects from a Schedule.
#pragma once

#include <string>
#include <utility>
#include <vector>

#include "deserve.h"
#include "pipeline.hpp"

namespace dsb {

struct GpuOptions {
    int device0 = 0;
    int n_devices = 0;         // 0 = all visible; stage s runs on device0 + s % n_devices
    bool real_delay = true;    // enforce the injected hop delay in wall time
    int64_t max_circuits = 0;  // execute only the first circuits of the schedule (0 = all)
    uint64_t weight_seed = 0x5EED0001ULL;
    bool collect_tokens = false;  // D2H the sampled ids of every circuit
    bool step_timing = true;      // CUDA events around every stage step
    bool trace = false;           // keep the virtual trace: session_trace() rebuilds it on the real clock
};

struct StageRunStats {
    int device = 0;
    int64_t computes = 0, topups = 0;
    int64_t swap_plan_bytes = 0, swap_in_bytes = 0, swap_out_bytes = 0;
    double busy_ms = 0, device_ms = 0;
    std::vector<std::pair<int64_t, double>> steps;  // (rows, ms) per stage step
    std::vector<double> gaps;  // ms between the end of the previous step and this one's start
    std::vector<double> ends;  // ms from the run's start to the end of each step (GPU events)
    std::string kernel_stats;                       // ds_stage_kernel_stats JSON
};

struct SwapPair {  // one schedule swap-in: plan bytes vs what moved (ds_swap_stats)
    int64_t plan = 0, slot_in = 0, migrated = 0, moved_out = 0;
};

struct GpuRunResult {
    int64_t circuits = 0, decode_tokens = 0, rows = 0, wall_us = 0, device_us = 0;
    int64_t launches = 0, d2h_bytes = 0, h2d_bytes = 0;
    int64_t swap_wait_us = 0;  // measured: GPU time computes waited for their swap-ins
    std::vector<std::vector<SwapPair>> swaps;  // per stage: every schedule swap-in, plan vs moved
    std::vector<int64_t> page_bytes;           // per stage
    std::vector<StageRunStats> stages;
    std::vector<std::vector<int32_t>> tokens;  // per circuit: sampled ids of its need_logits rows
    std::string error;
    std::string to_json() const;
};

struct Session;
// rank < 0: every stage in this process (stage s on device0 + s % n_devices, hops by peer copy).
// rank >= 0: only stage `rank` on device0, hops over NCCL (nccl_ids: world ncclUniqueIds).
Session* session_create(const Config& cfg, const Plan& plan, Schedule sched, const ds_model_desc& md,
                        const GpuOptions& opt, int rank = -1, int world = 1,
                        const void* nccl_ids = nullptr, std::vector<Record> vtrace = {});
GpuRunResult session_run(Session* s, bool profile, bool collect_tokens);
void session_destroy(Session* s);

// The last run's events on the real clock (reference EventTrace, trace.hpp:24-42): the virtual
// trace's events with the times the hardware produced them (GPU events mapped to the host
// steady clock, hop arrivals from the host), in (time, virtual seq) order. Only events of the
// stages this process runs and of the executed schedule prefix. t0_us: the steady-clock origin
// (< 0: this run's start). renumber = false keeps the virtual seq (for merging rank traces).
std::vector<Record> session_trace(Session* s, int64_t t0_us, bool renumber);
// later runs execute only the first max_circuits of the prepared prefix (0 = all of it)
void session_limit(Session* s, int64_t max_circuits);
int64_t session_t0(Session* s);  // steady-clock us of the last run's start
int64_t session_end(Session* s);  // us from t0 to the last run's end
const Config& session_config(Session* s);
const Plan& session_plan(Session* s);
int64_t session_vocab(Session* s);
// rows sampled for these requests are copied (fp32 logits) into a host pool at every run
void session_capture(Session* s, const std::vector<int64_t>& reqs);
// (circuit, req, position, row) of every captured row and the logits [n x vocab]
void session_captured(Session* s, std::vector<int64_t>* meta, const float** logits, int64_t* n);

GpuRunResult run_on_gpus(const Config& cfg, const Plan& plan, const Schedule& sched,
                         const ds_model_desc& md, const GpuOptions& opt);

}  // namespace dsb
