// Integer domain of the DeServe stage-step path: model/topology/workload specs, the planner's
// outputs, the event record, and the scheduler that drives the stages. Units follow the
// reference (include/pipesim/types.hpp:15-21): int64 bytes, int64 microseconds, int64 tokens,
// 256-token KV pages.
#pragma once

#include <cstdint>
#include <stdexcept>
#include <string>
#include <utility>
#include <vector>

namespace dsb {

using Bytes = int64_t;
using Micros = int64_t;
using Tokens = int64_t;

constexpr Tokens kPage = 256;  // reference kPageTokens (types.hpp:21)

inline int64_t div_up(int64_t a, int64_t b) { return (a + b - 1) / b; }
// round(a*num/den), half away from zero, a >= 0 (reference scale_round, types.hpp:28-30)
inline int64_t mul_div_round(int64_t a, int64_t num, int64_t den) {
    return (2 * a * num + den) / (2 * den);
}

struct ConfigError : std::runtime_error { using std::runtime_error::runtime_error; };
struct PlanError : std::runtime_error { using std::runtime_error::runtime_error; };
struct SimError : std::runtime_error { using std::runtime_error::runtime_error; };

struct CalPoint {
    int64_t batch;
    Micros us;
};
using Calibration = std::vector<CalPoint>;

struct Model {
    std::string name;
    int64_t num_layers = 0;
    Bytes weight_bytes_total = 0, embedding_bytes = 0, output_layer_bytes = 0;
    Bytes kv_bytes_per_token = 0;
    Tokens max_seq_len = 0;
    Bytes transformer_bytes() const { return weight_bytes_total - embedding_bytes - output_layer_bytes; }
    Bytes layer_range_bytes(int64_t b, int64_t e) const {
        const Bytes t = transformer_bytes();
        return t * e / num_layers - t * b / num_layers;
    }
};

struct Node {
    std::string id;
    Bytes mem = 0;
    Bytes pcie = 0;
    std::string cal_name;
    Calibration cal;
};

struct Link {
    std::string src, dst;
    Micros latency = 0;
    Bytes bw = 0;
};

struct Topo {
    std::vector<Node> nodes;
    std::vector<Link> links;
    const Node* node(const std::string& id) const;
    const Link* link(const std::string& s, const std::string& d) const;
};

struct Workload {
    Tokens prompt_min = 0, prompt_max = 0, output_min = 0, output_max = 0;
    int64_t concurrency = 0;
    int64_t duration_s = 0, warmup_s = 0;
    uint64_t seed = 0;
    std::string trace_path;
};

struct Policy {
    bool offload = true;
    int64_t nb_override = 0;
    int64_t prefill_chunk = 256;
    Bytes hidden_bytes_per_token = 16384;
    int64_t kv_reserve_permille = 300;
    int64_t calibration_ref_layers = 0;
    std::string ring_order = "config";
    int64_t pool_scale_milli = 1000;
    std::string pool_time_basis = "compute";
};

struct Budget {
    Bytes m_total = 0, m_weights = 0, m_kv = 0, m_global = 0;
    int64_t n_mb = 0;
    Bytes per_mb_plain = 0, per_mb_offload = 0;
    bool offload = false;
    Bytes per_mb() const { return offload ? per_mb_offload : per_mb_plain; }
    Bytes local_bytes() const { return per_mb() - m_global; }
};

struct StagePlanD {
    std::string node_id;
    int64_t layer_begin = 0, layer_end = 0;
    Bytes weight_bytes = 0;
    Bytes pcie = 0;
    Budget budget;
    int64_t batch = 0;
    Micros stage_time = 0;
};

struct Plan {
    std::vector<StagePlanD> stages;
    int64_t n_mb = 0;
    std::vector<Link> ring;
    Micros t_s = 0;
    bool offload = false;
    bool converged = true;
    int64_t iterations = 0;
    Tokens seq_budget = 0;
    Policy policy;
    int64_t S() const { return int64_t(stages.size()); }
    int64_t B() const { return stages.empty() ? 0 : stages.front().batch; }
    Micros hop_latency_sum() const {
        Micros s = 0;
        for (const auto& l : ring) s += l.latency;
        return s;
    }
    std::string to_json() const;
    static Plan from_json(const std::string& text);
};

// ---- perf model (reference src/perf_model.cpp)
void check_calibration(const Calibration& c);
const Calibration& table1();
Calibration read_calibration_csv(const std::string& path);
Micros compute_time(const Calibration& c, int64_t batch);
Micros stage_time(const Calibration& c, int64_t batch, int64_t layers, int64_t ref_layers);
Bytes page_size(const Model& m, int64_t layers, int64_t total_layers);
Bytes kv_size(const Model& m, Tokens tokens, int64_t layers, int64_t total_layers);
Bytes global_pool(Bytes pcie, Micros t, Bytes page);
Budget make_budget(const Node& n, Bytes weights, int64_t n_mb, Bytes m_global, bool offload);
int64_t batch_fit(Bytes budget, const Model& m, int64_t layers, int64_t total_layers, Tokens seq);

// ---- planner (reference src/planner.cpp)
std::vector<std::pair<int64_t, int64_t>> split_layers(const Model& m, const Topo& t,
                                                      const std::vector<std::string>& order,
                                                      int64_t reserve_permille);
int64_t bubble_free_nb(int64_t S, Micros t_s, Micros hop_sum);
std::vector<std::string> ring_order(const Topo& t, const std::string& mode);
Plan make_plan(const Model& m, const Topo& t, const Workload& w, const Policy& p);

// ---- config (reference src/config.cpp, same document format)
struct Config {
    Model model;
    Topo topo;
    Workload workload;
    Policy policy;
    std::vector<Micros> sweep_latencies;
    std::string dir;
};
Config parse_config(const std::string& text, const std::string& dir);
// policy name "baseline"|"offload"|"opt" (reference sweep.cpp:26-43); empty = unchanged
Policy apply_policy_name(const Policy& base, const std::string& name, int64_t n_stages);

// ---- events (reference include/pipesim/trace.hpp)
enum class Ev : uint8_t { ComputeStart, ComputeEnd, TransferArrive, SwapInDone, SwapOutDone, RequestAdmit, RequestComplete };
const char* ev_name(Ev k);

struct Record {
    Micros t = 0;
    int64_t seq = 0;
    Ev kind = Ev::ComputeStart;
    int32_t stage = -1, mb = -1;
    int64_t a = 0, b = 0, c = 0;
};
std::string trace_text(const std::vector<Record>& tr);
// reference read_trace (src/trace.cpp:54-88); throws ConfigError on a malformed line
std::vector<Record> parse_trace(const std::string& text);
// SimReport fields (reference build_report, src/sim.cpp:501-532) recomputed from a trace over
// [w0, w1): tokens as windowed_stats (src/workload.cpp:82-116), busy = compute intervals,
// stall = the part of a swap-dependent compute's wait (stage free and microbatch arrived) that
// its SwapInDone covers, as the engine's stall_acc (src/sim.cpp:355-382).
struct Report;
Report report_from_trace(const std::vector<Record>& tr, int64_t n_stages, Micros w0, Micros w1,
                         uint64_t seed);
struct Plan;
Report report_from_json(const std::string& text);
// reference report_to_kv (src/sweep.cpp:146-195) and SweepResult::to_csv (sweep.cpp:68-82)
std::string report_kv(const Report& r, const Plan& p, Micros latency, const std::string& policy);
std::string sweep_csv(const std::vector<Micros>& lat, const std::vector<std::string>& pol,
                      const std::vector<double>& tput);

// ---- profit model on reports (economics.cpp; reference economics.cpp:9-81, config.cpp:169-199)
struct Pricing {
    std::string name;
    int64_t cost_per_hour_micro = 0;  // C
    int64_t price_nano = 0;           // P (unified price per token)
    int64_t price_in_nano = 0;        // P_I
    int64_t price_out_nano = 0;       // P_O
    bool unified() const { return price_in_nano == price_nano && price_out_nano == price_nano; }
};
struct Profit {
    int64_t revenue_micro = 0, cost_micro = 0, profit_micro = 0;
    double min_throughput = 0, achieved_throughput = 0;
    bool profitable = false;
};
// the config's "pricing" object ({"preset": name} or money fields); throws ConfigError
Pricing parse_pricing(const std::string& json_text);
Profit analyze(const Report& r, const Pricing& p);
// the pricing block report_to_kv appends (src/sweep.cpp:187-194)
std::string profit_kv(const Profit& p);

struct StageStats {
    Micros busy = 0, stall = 0, bubble = 0;
    double busy_frac = 0, stall_frac = 0, bubble_frac = 0;
};
struct Report {
    Micros w0 = 0, w1 = 0;
    Tokens n_in = 0, n_out = 0;
    double wall_s = 0, in_tps = 0, out_tps = 0, total_tps = 0;
    std::vector<StageStats> stages;
    double mean_bubble = 0, max_bubble = 0;
    Micros swap_stall = 0;
    int64_t completed = 0, live = 0, admitted = 0;
    uint64_t seed = 0;
    std::string to_json() const;
};

// ---- the schedule the GPU executor replays
struct RowSpec {
    int32_t slot;
    int32_t pos;
    int32_t n_tok;
    int32_t need_logits;
    int32_t is_decode;
    int64_t req;
};
struct Circuit {
    int32_t mb = 0;
    int64_t eff_batch = 0, n_decode = 0;
    std::vector<RowSpec> rows;
    std::vector<int32_t> completed_slots;  // slots whose requests finished at this circuit's end
    Micros t_end = -1;                     // virtual time of the circuit end (last stage)
    // the circuit whose last-stage end sent this microbatch to stage 0 (its own previous circuit
    // via send_onward, or another microbatch's via wake_parked; -1 = placed at t=0) and the
    // payload of that hop (reference sim.cpp:277-294,430-439)
    int64_t trig = -1;
    Bytes trig_payload = 0;
};
enum class OpKind : uint8_t { Compute, SwapIn, Release };
struct StageOp {
    OpKind kind;
    int32_t mb;
    int32_t slot;        // SwapIn: global slot; Release: request slot
    int64_t circuit;     // Compute: circuit index
    int64_t plan_bytes;  // SwapIn: reference global_portion bytes
    Micros t;            // virtual issue time
    int64_t evict_bytes = 0;  // SwapIn: bytes of the slot occupant's eviction (SwapOutDone b)
};
struct Schedule {
    std::vector<Circuit> circuits;
    std::vector<std::vector<StageOp>> ops;  // per stage, in issue order
};

struct SimOutput {
    Report report;
    std::vector<Record> trace;
    Schedule schedule;
};

// Virtual-clock execution of a plan (reference Engine, src/sim.cpp:95-587). Stage durations come
// from the node calibration exactly as scaled_stage_time; the output trace is byte-identical to
// the reference's. Throws SimError on plan/topology mismatch or deadlock.
SimOutput simulate(const Plan& plan, const Topo& topo, const Workload& wl, const Model& model,
                   bool keep_trace = true, bool keep_schedule = false);
double analytic_throughput(const Plan& plan);
// lengths of request `index` under the workload's SplitMix64 stream (reference workload.cpp:36-53)
std::pair<Tokens, Tokens> request_lengths(const Workload& w, int64_t index);  // reference steady_state_throughput (sim.cpp:597-604)

}  // namespace dsb
