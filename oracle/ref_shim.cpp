// TEST INFRASTRUCTURE ONLY — never linked into the product.
//
// extern "C" shim over the UNMODIFIED reference sources (/root/reference/proj/src, compiled by
// oracle/Makefile into oracle/_ref/libpipesim_ref.so). Tests, __graft_entry__.smoke() and the
// cpu_baseline / --impl reference legs of bench.py call it as the integer oracle:
//   plan()                 src/planner.cpp:140-276
//   run() / Engine         src/sim.cpp:534-595
//   replay_check           src/sim.cpp:606-697
//   windowed_stats         src/workload.cpp:82-116
//   perf-model functions   src/perf_model.cpp:85-175
#include <cstring>
#include <fstream>
#include <sstream>
#include <string>

#include "pipesim/config.hpp"
#include "pipesim/economics.hpp"
#include "pipesim/perf_model.hpp"
#include "pipesim/planner.hpp"
#include "pipesim/sim.hpp"
#include "pipesim/sweep.hpp"
#include "pipesim/trace.hpp"
#include "pipesim/workload.hpp"

using namespace pipesim;

namespace {
thread_local std::string g_err;

void put(const std::string& s, char* out, size_t cap) {
    if (!out || !cap) return;
    const size_t n = std::min(cap - 1, s.size());
    std::memcpy(out, s.data(), n);
    out[n] = 0;
}

std::string report_json(const SimReport& r) {
    std::ostringstream os;
    os.precision(17);
    os << "{\"window_start_us\":" << r.window_start_us << ",\"window_end_us\":" << r.window_end_us
       << ",\"input_tokens\":" << r.input_tokens << ",\"output_tokens\":" << r.output_tokens
       << ",\"wall_time_s\":" << r.wall_time_s << ",\"input_throughput\":" << r.input_throughput
       << ",\"output_throughput\":" << r.output_throughput
       << ",\"total_throughput\":" << r.total_throughput
       << ",\"mean_bubble_fraction\":" << r.mean_bubble_fraction
       << ",\"max_bubble_fraction\":" << r.max_bubble_fraction << ",\"swap_stall_us\":" << r.swap_stall_us
       << ",\"completed_requests\":" << r.completed_requests << ",\"live_requests\":" << r.live_requests
       << ",\"admitted_requests\":" << r.admitted_requests << ",\"rng_seed\":" << r.rng_seed
       << ",\"stages\":[";
    for (size_t i = 0; i < r.stages.size(); ++i) {
        const auto& s = r.stages[i];
        os << (i ? "," : "") << "{\"busy_us\":" << s.busy_us << ",\"stall_us\":" << s.stall_us
           << ",\"bubble_us\":" << s.bubble_us << ",\"busy_fraction\":" << s.busy_fraction
           << ",\"transfer_wait_fraction\":" << s.transfer_wait_fraction
           << ",\"bubble_fraction\":" << s.bubble_fraction << "}";
    }
    os << "]}";
    return os.str();
}

struct Planned {
    RunConfig cfg;
    Topology topo;
    PipelinePlan plan;
};

Planned make(const char* text, const char* dir, const char* policy, long long latency, long long nb) {
    Planned p;
    p.cfg = parse_config(text, dir ? dir : "");
    p.topo = latency >= 0 ? with_uniform_latency(p.cfg.topology, latency) : p.cfg.topology;
    SchedulerPolicy pol = p.cfg.scheduler;
    if (policy && *policy)
        pol = apply_policy(pol, policy_from_name(policy), int64_t(p.cfg.topology.nodes.size()));
    if (nb >= 0) pol.nb_override = nb;
    p.plan = plan(p.cfg.model, p.topo, p.cfg.workload, pol);
    return p;
}

template <class F>
int guard(F&& f) {
    try {
        return f();
    } catch (const std::exception& e) {
        g_err = e.what();
        return 1;
    }
}
}  // namespace

extern "C" {

const char* ref_last_error() { return g_err.c_str(); }

int ref_plan_config(const char* text, const char* dir, const char* policy, long long latency,
                    long long nb, char* out, size_t cap) {
    return guard([&] {
        put(make(text, dir, policy, latency, nb).plan.to_json(), out, cap);
        return 0;
    });
}

int ref_sim_config(const char* text, const char* dir, const char* policy, long long latency,
                   long long nb, const char* trace_path, char* report, size_t cap) {
    return guard([&] {
        Planned p = make(text, dir, policy, latency, nb);
        SimResult r = run(p.plan, p.topo, p.cfg.workload, p.cfg.model);
        if (trace_path && *trace_path) write_trace_file(trace_path, r.trace);
        put(report_json(r.report), report, cap);
        return 0;
    });
}

// report_to_kv (src/sweep.cpp:146-195) of run() on the config (policy/latency as ref_plan_config)
int ref_report_kv(const char* text, const char* dir, const char* policy, long long latency,
                  long long nb, char* out, size_t cap) {
    return guard([&] {
        Planned p = make(text, dir, policy, latency, nb);
        SimResult r = run(p.plan, p.topo, p.cfg.workload, p.cfg.model);
        const Micros lat = p.topo.links.empty() ? 0 : p.topo.links.front().latency_us;
        put(report_to_kv(r.report, p.plan, lat, policy && *policy ? policy : "config", nullptr), out, cap);
        return 0;
    });
}

// report_to_kv with the config's pricing (analyze, src/economics.cpp:21-59): the reference's
// priced report.kv of run() on the config; pricing_json (optional) replaces the config's section
int ref_report_kv_priced(const char* text, const char* dir, const char* policy, long long latency,
                         long long nb, char* out, size_t cap) {
    return guard([&] {
        Planned p = make(text, dir, policy, latency, nb);
        if (!p.cfg.has_pricing) throw ConfigError("config has no pricing section");
        SimResult r = run(p.plan, p.topo, p.cfg.workload, p.cfg.model);
        const Micros lat = p.topo.links.empty() ? 0 : p.topo.links.front().latency_us;
        const ProfitAnalysis pa = analyze(r.report, p.cfg.pricing);
        put(report_to_kv(r.report, p.plan, lat, policy && *policy ? policy : "config", &pa), out, cap);
        return 0;
    });
}

// run_sweep(...).to_csv() (src/sweep.cpp:68-82,101-144) over the config's sweep latencies
int ref_sweep_csv(const char* text, const char* dir, char* out, size_t cap) {
    return guard([&] {
        RunConfig cfg = parse_config(text, dir ? dir : "");
        SweepResult r = run_sweep(cfg, {Policy::Baseline, Policy::Offload, Policy::Opt}, 1, false);
        put(r.to_csv(), out, cap);
        return 0;
    });
}

int ref_sim_plan(const char* text, const char* dir, const char* plan_json, const char* trace_path,
                 char* report, size_t cap) {
    return guard([&] {
        RunConfig cfg = parse_config(text, dir ? dir : "");
        PipelinePlan p = PipelinePlan::from_json(plan_json);
        SimResult r = run(p, cfg.topology, cfg.workload, cfg.model);
        if (trace_path && *trace_path) write_trace_file(trace_path, r.trace);
        put(report_json(r.report), report, cap);
        return 0;
    });
}

int ref_stage_time(const long long* b, const long long* t, long long n, long long batch,
                   long long layers, long long ref_layers, long long* out) {
    return guard([&] {
        CalibrationTable c;
        for (long long i = 0; i < n; ++i) c.entries.push_back({b[i], t[i]});
        *out = scaled_stage_time(c, batch, layers, ref_layers);
        return 0;
    });
}

int ref_page_bytes(long long kv_per_token, long long layers, long long total, long long* out) {
    return guard([&] {
        ModelSpec m;
        m.kv_bytes_per_token = kv_per_token;
        *out = page_bytes(m, {layers, total});
        return 0;
    });
}

int ref_global_pool_size(long long w, long long t, long long page, long long* out) {
    return guard([&] {
        *out = global_pool_size(w, t, page);
        return 0;
    });
}

// out: m_kv, m_global, per_mb_no_offload, per_mb_offload, local_pool
int ref_memory_budget(long long mem, long long weights, long long nb, long long mg, int offload,
                      long long* out) {
    return guard([&] {
        NodeSpec n;
        n.node_id = "n";
        n.gpu_mem_bytes = mem;
        MemoryBudget b = memory_budget(n, weights, nb, mg, offload != 0);
        out[0] = b.m_kv;
        out[1] = b.m_global_pool;
        out[2] = b.m_per_microbatch_no_offload;
        out[3] = b.m_per_microbatch_offload;
        out[4] = b.local_pool_bytes();
        return 0;
    });
}

// violations as "kind entity\n" lines
int ref_replay_check(const char* trace_path, const char* plan_json, char* out, size_t cap) {
    return guard([&] {
        EventTrace t = read_trace_file(trace_path);
        PipelinePlan p = PipelinePlan::from_json(plan_json);
        std::string s;
        for (const auto& v : replay_check(t, p)) s += v.kind + " " + v.entity + "\n";
        put(s, out, cap);
        return 0;
    });
}

int ref_windowed_stats(const char* trace_path, long long start, long long end, int completed_based,
                       long long* out) {
    return guard([&] {
        EventTrace t = read_trace_file(trace_path);
        WindowStats w = completed_based ? windowed_stats_completed(t, start, end)
                                        : windowed_stats(t, start, end);
        out[0] = w.input_tokens;
        out[1] = w.output_tokens;
        out[2] = w.window_us;
        return 0;
    });
}

double ref_steady_state(const char* plan_json) {
    try {
        return steady_state_throughput(PipelinePlan::from_json(plan_json));
    } catch (const std::exception& e) {
        g_err = e.what();
        return -1;
    }
}

int ref_request(unsigned long long seed, long long pmin, long long pmax, long long omin,
                long long omax, long long index, long long* out) {
    return guard([&] {
        WorkloadSpec w;
        w.rng_seed = seed;
        w.prompt_len_min = pmin;
        w.prompt_len_max = pmax;
        w.output_len_min = omin;
        w.output_len_max = omax;
        Request r = RequestGenerator(w).make(index);
        out[0] = r.prompt_len;
        out[1] = r.target_output_len;
        return 0;
    });
}

}  // extern "C"
