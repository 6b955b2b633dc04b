// The reference-side binding a pipesim maintainer adds to run a config on B200s (INTEGRATION.md
// section 1): the same signature shape as pipesim::run() (include/pipesim/sim.hpp:47-55), returning
// a pipesim::SimResult built from ds_run's real-clock EventTrace (read back with the reference's
// own read_trace_file, src/trace.cpp:54-88) and its SimReport fields. Compiled against the
// UNMODIFIED reference headers + libpipesim (oracle/Makefile, target `binding`), linked with
// libdeserve_b200.so; used by tests/test_gpu_trace.py to run the reference's replay_check and
// windowed_stats in C++ on a hardware run. Test/integration code: not part of the product library.
#include <cstdio>
#include <stdexcept>
#include <string>
#include <vector>

#include "deserve.h"
#include "json.hpp"
#include "pipesim/sim.hpp"
#include "pipesim/trace.hpp"
#include "pipesim/workload.hpp"

namespace pipesim_b200 {

pipesim::SimResult run_on_b200(const std::string& config_json, const std::string& config_dir,
                               const ds_model_desc& dims, const ds_gpu_opts& opts,
                               const std::string& trace_path) {
    std::vector<char> buf(size_t(64) << 20);
    size_t need = 0;
    const ds_status st = ds_run(config_json.c_str(), config_dir.c_str(), "", -1, -1, &dims, &opts,
                                trace_path.c_str(), buf.data(), buf.size(), &need);
    if (st == DS_ERR_ARG) throw pipesim::ConfigError(ds_last_error());
    if (st == DS_ERR_PLAN) throw pipesim::PlanError(ds_last_error());
    if (st != DS_OK) throw pipesim::SimError(ds_last_error());
    const auto j = nlohmann::json::parse(buf.data()).at("report");
    pipesim::SimResult r;
    pipesim::SimReport& rep = r.report;
    rep.window_start_us = j.at("window_start_us");
    rep.window_end_us = j.at("window_end_us");
    rep.input_tokens = j.at("input_tokens");
    rep.output_tokens = j.at("output_tokens");
    rep.wall_time_s = j.at("wall_time_s");
    rep.input_throughput = j.at("input_throughput");
    rep.output_throughput = j.at("output_throughput");
    rep.total_throughput = j.at("total_throughput");
    rep.mean_bubble_fraction = j.at("mean_bubble_fraction");
    rep.max_bubble_fraction = j.at("max_bubble_fraction");
    rep.swap_stall_us = j.at("swap_stall_us");
    rep.completed_requests = j.at("completed_requests");
    rep.live_requests = j.at("live_requests");
    rep.admitted_requests = j.at("admitted_requests");
    rep.rng_seed = j.at("rng_seed");
    for (const auto& s : j.at("stages")) {
        pipesim::StageMetrics m;
        m.busy_us = s.at("busy_us");
        m.stall_us = s.at("stall_us");
        m.bubble_us = s.at("bubble_us");
        m.busy_fraction = s.at("busy_fraction");
        m.transfer_wait_fraction = s.at("transfer_wait_fraction");
        m.bubble_fraction = s.at("bubble_fraction");
        rep.stages.push_back(m);
    }
    r.trace = pipesim::read_trace_file(trace_path);
    return r;
}

}  // namespace pipesim_b200

// C entry for the tests: runs the config on the GPU through the binding, then the reference's
// replay_check (against the reference planner's plan of the same config) and windowed_stats on
// the returned SimResult. out: {"violations", "trace_events", "report_output_tokens",
// "windowed_output_tokens", "output_throughput"}.
extern "C" int b200_run_and_check(const char* config_json, const char* config_dir, const char* plan_json,
                                  const ds_model_desc* dims, const ds_gpu_opts* opts,
                                  const char* trace_path, char* out, size_t cap) {
    try {
        pipesim::SimResult r = pipesim_b200::run_on_b200(config_json, config_dir, *dims, *opts, trace_path);
        const pipesim::PipelinePlan plan = pipesim::PipelinePlan::from_json(plan_json);
        const auto viol = pipesim::replay_check(r.trace, plan);
        const auto w = pipesim::windowed_stats(r.trace, r.report.window_start_us, r.report.window_end_us);
        nlohmann::json o;
        o["violations"] = viol.size();
        o["trace_events"] = r.trace.size();
        o["report_output_tokens"] = r.report.output_tokens;
        o["windowed_output_tokens"] = w.output_tokens;
        o["output_throughput"] = r.report.output_throughput;
        const std::string s = o.dump();
        snprintf(out, cap, "%s", s.c_str());
        return 0;
    } catch (const std::exception& e) {
        snprintf(out, cap, "error: %s", e.what());
        return 1;
    }
}
