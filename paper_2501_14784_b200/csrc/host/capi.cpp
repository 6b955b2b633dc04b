// C ABI for the integer half of the path (include/deserve.h): perf model, planner and the
// virtual-clock scheduler. Exceptions never cross the boundary; they become ds_status codes
// with a thread-local message (ConfigError -> DS_ERR_ARG, PlanError -> DS_ERR_PLAN,
// SimError/other -> DS_ERR_RUNTIME; reference exit-code mapping cli.cpp:219-231).
#include <cstring>
#include <fstream>
#include <string>

#include "capi_util.hpp"
#include "pipeline.hpp"

namespace {
thread_local std::string g_last_error;

template <class F>
ds_status guarded(F&& f) {
    try {
        return f();
    } catch (const dsb::ConfigError& e) {
        return ds_fail(DS_ERR_ARG, e.what());
    } catch (const dsb::PlanError& e) {
        return ds_fail(DS_ERR_PLAN, e.what());
    } catch (const std::invalid_argument& e) {
        return ds_fail(DS_ERR_ARG, e.what());
    } catch (const std::exception& e) {
        return ds_fail(DS_ERR_RUNTIME, e.what());
    }
}

void copy_out(const std::string& s, char* out, size_t cap, size_t* needed) {
    if (needed) *needed = s.size() + 1;
    if (out && cap) {
        const size_t n = std::min(cap - 1, s.size());
        std::memcpy(out, s.data(), n);
        out[n] = 0;
    }
}
}  // namespace

int32_t ds_fail(int32_t code, const std::string& msg) {
    g_last_error = msg;
    return code;
}

namespace dsb {
// Shared by the C ABI and the GPU executor: config text -> (config, plan) with overrides.
std::pair<Config, Plan> plan_from_config(const char* json_text, const char* dir, const char* policy,
                                         int64_t latency_us, int64_t nb_override) {
    Config c = parse_config(json_text ? json_text : "", dir ? dir : "");
    if (latency_us >= 0)
        for (auto& l : c.topo.links) l.latency = latency_us;
    c.policy = apply_policy_name(c.policy, policy ? policy : "", int64_t(c.topo.nodes.size()));
    if (nb_override >= 0) c.policy.nb_override = nb_override;
    Plan p = make_plan(c.model, c.topo, c.workload, c.policy);
    return {std::move(c), std::move(p)};
}
}  // namespace dsb

extern "C" {

const char* ds_last_error(void) { return g_last_error.c_str(); }
const char* ds_version(void) { return "deserve-b200 0.1 (sm_100a)"; }

int32_t ds_prompt_token_id(int64_t req_id, int32_t pos) { return ds_prompt_token(req_id, pos); }

ds_status ds_stage_time_us(const int64_t* batch_sizes, const int64_t* times_us, int64_t n,
                           int64_t batch, int64_t layers, int64_t ref_layers, int64_t* out_us) {
    return guarded([&] {
        if (!batch_sizes || !times_us || !out_us || n < 0) return ds_fail(DS_ERR_ARG, "null argument");
        dsb::Calibration c;
        for (int64_t i = 0; i < n; ++i) c.push_back({batch_sizes[i], times_us[i]});
        *out_us = dsb::stage_time(c, batch, layers, ref_layers);
        return DS_OK;
    });
}

ds_status ds_page_bytes(int64_t kv_bytes_per_token, int64_t layers, int64_t total_layers, int64_t* out) {
    return guarded([&] {
        dsb::Model m;
        m.kv_bytes_per_token = kv_bytes_per_token;
        *out = dsb::page_size(m, layers, total_layers);
        return DS_OK;
    });
}

ds_status ds_global_pool_size(int64_t pcie_bw, int64_t stage_time_us, int64_t page, int64_t* out) {
    return guarded([&] {
        *out = dsb::global_pool(pcie_bw, stage_time_us, page);
        return DS_OK;
    });
}

ds_status ds_memory_budget(int64_t mem, int64_t weights, int64_t n_mb, int64_t m_global,
                           int32_t offload, int64_t* out5) {
    return guarded([&] {
        dsb::Node n;
        n.id = "node";
        n.mem = mem;
        const dsb::Budget b = dsb::make_budget(n, weights, n_mb, m_global, offload != 0);
        out5[0] = b.m_kv;
        out5[1] = b.m_global;
        out5[2] = b.per_mb_plain;
        out5[3] = b.per_mb_offload;
        out5[4] = b.local_bytes();
        return DS_OK;
    });
}

ds_status ds_request_lengths(uint64_t seed, int64_t prompt_min, int64_t prompt_max, int64_t output_min,
                             int64_t output_max, int64_t index, int64_t* out2) {
    return guarded([&] {
        dsb::Workload w;
        w.seed = seed;
        w.prompt_min = prompt_min;
        w.prompt_max = prompt_max;
        w.output_min = output_min;
        w.output_max = output_max;
        const auto pr = dsb::request_lengths(w, index);
        out2[0] = pr.first;
        out2[1] = pr.second;
        return DS_OK;
    });
}

ds_status ds_steady_state_throughput(const char* plan_json, double* out) {
    return guarded([&] {
        *out = dsb::analytic_throughput(dsb::Plan::from_json(plan_json ? plan_json : ""));
        return DS_OK;
    });
}

ds_status ds_plan_config(const char* config_json, const char* config_dir, const char* policy,
                         int64_t latency_us, int64_t nb_override, char* out, size_t cap,
                         size_t* needed) {
    return guarded([&] {
        auto cp = dsb::plan_from_config(config_json, config_dir, policy, latency_us, nb_override);
        copy_out(cp.second.to_json(), out, cap, needed);
        return DS_OK;
    });
}

ds_status ds_sim_config(const char* config_json, const char* config_dir, const char* policy,
                        int64_t latency_us, int64_t nb_override, const char* trace_path,
                        char* report_json, size_t cap) {
    return guarded([&] {
        auto cp = dsb::plan_from_config(config_json, config_dir, policy, latency_us, nb_override);
        const bool want_trace = trace_path && *trace_path;
        dsb::SimOutput o = dsb::simulate(cp.second, cp.first.topo, cp.first.workload, cp.first.model,
                                         want_trace, false);
        if (want_trace) {
            std::ofstream f(trace_path, std::ios::binary);
            if (!f) return ds_fail(DS_ERR_RUNTIME, std::string("cannot write trace file ") + trace_path);
            const std::string t = dsb::trace_text(o.trace);
            f.write(t.data(), std::streamsize(t.size()));
        }
        copy_out(o.report.to_json(), report_json, cap, nullptr);
        return DS_OK;
    });
}

ds_status ds_sim_plan(const char* config_json, const char* config_dir, const char* plan_json,
                      const char* trace_path, char* report_json, size_t cap) {
    return guarded([&] {
        dsb::Config c = dsb::parse_config(config_json ? config_json : "", config_dir ? config_dir : "");
        dsb::Plan p = dsb::Plan::from_json(plan_json ? plan_json : "");
        const bool want_trace = trace_path && *trace_path;
        dsb::SimOutput o = dsb::simulate(p, c.topo, c.workload, c.model, want_trace, false);
        if (want_trace) {
            std::ofstream f(trace_path, std::ios::binary);
            if (!f) return ds_fail(DS_ERR_RUNTIME, std::string("cannot write trace file ") + trace_path);
            const std::string t = dsb::trace_text(o.trace);
            f.write(t.data(), std::streamsize(t.size()));
        }
        copy_out(o.report.to_json(), report_json, cap, nullptr);
        return DS_OK;
    });
}

}  // extern "C"
