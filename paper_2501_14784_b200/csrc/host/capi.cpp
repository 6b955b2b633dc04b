// C ABI for the integer half of the path (include/deserve.h): perf model, planner and the
// virtual-clock scheduler. Exceptions never cross the boundary; they become ds_status codes
// with a thread-local message (ConfigError -> DS_ERR_ARG, PlanError -> DS_ERR_PLAN,
// SimError/other -> DS_ERR_RUNTIME; reference exit-code mapping cli.cpp:219-231).
#include <algorithm>
#include <cstring>
#include <fstream>
#include <sstream>
#include <string>

#include "capi_util.hpp"
#include "executor.hpp"
#include "hop_nccl.hpp"
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

ds_status ds_schedule_config(const char* config_json, const char* config_dir, const char* policy,
                             int64_t latency_us, int64_t nb_override, int64_t max_circuits, char* out,
                             size_t cap, size_t* needed) {
    return guarded([&] {
        auto cp = dsb::plan_from_config(config_json, config_dir, policy, latency_us, nb_override);
        dsb::SimOutput o = dsb::simulate(cp.second, cp.first.topo, cp.first.workload, cp.first.model,
                                         false, true);
        const dsb::Schedule& sc = o.schedule;
        const int64_t n = max_circuits > 0 ? std::min<int64_t>(max_circuits, sc.circuits.size())
                                           : int64_t(sc.circuits.size());
        std::string js = "{\"circuits\":[";
        for (int64_t c = 0; c < n; ++c) {
            const auto& ci = sc.circuits[c];
            js += (c ? ",{" : "{") + std::string("\"mb\":") + std::to_string(ci.mb) +
                  ",\"eff_batch\":" + std::to_string(ci.eff_batch) + ",\"n_decode\":" +
                  std::to_string(ci.n_decode) + ",\"t_end\":" + std::to_string(ci.t_end) +
                  ",\"trig\":" + std::to_string(ci.trig) + ",\"trig_payload\":" +
                  std::to_string(ci.trig_payload) + ",\"rows\":[";
            for (size_t k = 0; k < ci.rows.size(); ++k) {
                const auto& r = ci.rows[k];
                js += (k ? ",[" : "[") + std::to_string(r.slot) + "," + std::to_string(r.pos) + "," +
                      std::to_string(r.n_tok) + "," + std::to_string(r.need_logits) + "," +
                      std::to_string(r.is_decode) + "," + std::to_string(r.req) + "]";
            }
            js += "],\"completed\":[";
            for (size_t k = 0; k < ci.completed_slots.size(); ++k)
                js += (k ? "," : "") + std::to_string(ci.completed_slots[k]);
            js += "]}";
        }
        js += "],\"ops\":[";
        for (size_t s = 0; s < sc.ops.size(); ++s) {
            js += s ? ",[" : "[";
            bool first = true;
            for (const auto& op : sc.ops[s]) {
                if (op.kind == dsb::OpKind::Compute && op.circuit >= n) break;
                js += (first ? "[" : ",[") + std::to_string(int(op.kind)) + "," + std::to_string(op.mb) +
                      "," + std::to_string(op.slot) + "," + std::to_string(op.circuit) + "," +
                      std::to_string(op.plan_bytes) + "," + std::to_string(op.t) + "," +
                      std::to_string(op.evict_bytes) + "]";
                first = false;
            }
            js += "]";
        }
        js += "]}";
        copy_out(js, out, cap, needed);
        return DS_OK;
    });
}

struct ds_session {
    dsb::Session* s = nullptr;
};

ds_status ds_session_create(const char* config_json, const char* config_dir, const char* policy,
                            int64_t latency_us, int64_t nb_override, const ds_model_desc* model,
                            const ds_gpu_opts* opts, ds_session** out) {
    return guarded([&] {
        if (!model || !opts || !out) return ds_fail(DS_ERR_ARG, "null argument");
        auto cp = dsb::plan_from_config(config_json, config_dir, policy, latency_us, nb_override);
        dsb::SimOutput o = dsb::simulate(cp.second, cp.first.topo, cp.first.workload, cp.first.model,
                                         opts->trace != 0, true);
        dsb::GpuOptions g;
        g.device0 = opts->device0;
        g.n_devices = opts->n_devices;
        g.real_delay = opts->real_delay != 0;
        g.collect_tokens = opts->collect_tokens != 0;
        g.max_circuits = opts->max_circuits;
        g.weight_seed = opts->weight_seed;
        g.trace = opts->trace != 0;
        ds_session* h = new ds_session();
        try {
            h->s = dsb::session_create(cp.first, cp.second, std::move(o.schedule), *model, g, -1, 1,
                                       nullptr, std::move(o.trace));
        } catch (...) {
            delete h;
            throw;
        }
        *out = h;
        return DS_OK;
    });
}

ds_status ds_nccl_unique_id(uint8_t* out128) {
    return guarded([&] {
        std::string why;
        const dsb::NcclApi* api = dsb::nccl_api(&why);
        if (!api) return ds_fail(DS_ERR_RUNTIME, "NCCL unavailable: " + why);
        ncclUniqueId id;
        if (api->GetUniqueId(&id) != ncclSuccess) return ds_fail(DS_ERR_RUNTIME, "ncclGetUniqueId failed");
        std::memcpy(out128, &id, sizeof(id));
        return DS_OK;
    });
}

ds_status ds_session_create_rank(const char* config_json, const char* config_dir, const char* policy,
                                 int64_t latency_us, int64_t nb_override, const ds_model_desc* model,
                                 const ds_gpu_opts* opts, int32_t rank, int32_t world,
                                 const uint8_t* nccl_ids, ds_session** out) {
    return guarded([&] {
        if (!model || !opts || !out || rank < 0 || world < 1) return ds_fail(DS_ERR_ARG, "bad argument");
        if (world > 1 && !nccl_ids) return ds_fail(DS_ERR_ARG, "nccl ids required for world > 1");
        auto cp = dsb::plan_from_config(config_json, config_dir, policy, latency_us, nb_override);
        dsb::SimOutput o = dsb::simulate(cp.second, cp.first.topo, cp.first.workload, cp.first.model,
                                         opts->trace != 0, true);
        dsb::GpuOptions g;
        g.device0 = opts->device0;
        g.n_devices = 1;
        g.real_delay = opts->real_delay != 0;
        g.collect_tokens = opts->collect_tokens != 0;
        g.max_circuits = opts->max_circuits;
        g.weight_seed = opts->weight_seed;
        g.trace = opts->trace != 0;
        ds_session* h = new ds_session();
        try {
            h->s = dsb::session_create(cp.first, cp.second, std::move(o.schedule), *model, g, rank, world,
                                       nccl_ids, std::move(o.trace));
        } catch (...) {
            delete h;
            throw;
        }
        *out = h;
        return DS_OK;
    });
}

ds_status ds_session_run(ds_session* h, int32_t profile, int32_t collect_tokens, char* report_json,
                         size_t cap, size_t* needed) {
    return guarded([&] {
        if (!h || !h->s) return ds_fail(DS_ERR_ARG, "null session");
        dsb::GpuRunResult r = dsb::session_run(h->s, profile != 0, collect_tokens != 0);
        copy_out(r.to_json(), report_json, cap, needed);
        if (!r.error.empty()) return ds_fail(DS_ERR_RUNTIME, r.error);
        return DS_OK;
    });
}

namespace {
std::string read_file(const char* path) {
    std::ifstream f(path, std::ios::binary);
    if (!f) throw dsb::ConfigError(std::string("cannot read ") + path);
    std::ostringstream os;
    os << f.rdbuf();
    return os.str();
}

void write_file(const char* path, const std::string& text) {
    std::ofstream f(path, std::ios::binary);
    if (!f) throw dsb::SimError(std::string("cannot write trace file ") + path);
    f.write(text.data(), std::streamsize(text.size()));
}

// report window of a hardware run: the workload's [warmup, duration) clipped to the run
std::pair<int64_t, int64_t> run_window(dsb::Session* s, int64_t w0, int64_t w1) {
    const dsb::Workload& wl = dsb::session_config(s).workload;
    if (w0 < 0) w0 = wl.warmup_s * 1'000'000;
    if (w1 < 0) w1 = std::min<int64_t>(wl.duration_s * 1'000'000, dsb::session_end(s) + 1);
    return {w0, w1};
}

std::string trace_report_json(dsb::Session* s, const std::vector<dsb::Record>& tr, int64_t w0, int64_t w1) {
    const auto win = run_window(s, w0, w1);
    const dsb::Plan& p = dsb::session_plan(s);
    dsb::Report r = dsb::report_from_trace(tr, p.S(), win.first, win.second, dsb::session_config(s).workload.seed);
    int64_t computes = 0;
    for (const auto& e : tr) computes += e.kind == dsb::Ev::ComputeStart;
    std::string js = r.to_json();
    js.pop_back();
    js += ",\"trace_events\":" + std::to_string(tr.size()) + ",\"trace_computes\":" + std::to_string(computes) +
          ",\"run_end_us\":" + std::to_string(dsb::session_end(s)) + "}";
    return js;
}
}  // namespace

ds_status ds_session_trace(ds_session* h, const char* trace_path, int64_t t0_us, int32_t keep_virtual_seq,
                           int64_t w0_us, int64_t w1_us, char* report_json, size_t cap, size_t* needed) {
    return guarded([&] {
        if (!h || !h->s) return ds_fail(DS_ERR_ARG, "null session");
        const std::vector<dsb::Record> tr = dsb::session_trace(h->s, t0_us, keep_virtual_seq == 0);
        if (trace_path && *trace_path) write_file(trace_path, dsb::trace_text(tr));
        copy_out(trace_report_json(h->s, tr, w0_us, w1_us), report_json, cap, needed);
        return DS_OK;
    });
}

ds_status ds_trace_merge(const char* const* paths, int32_t n, const char* out_path) {
    return guarded([&] {
        if (!paths || n < 1 || !out_path) return ds_fail(DS_ERR_ARG, "bad merge arguments");
        std::vector<dsb::Record> all;
        for (int32_t i = 0; i < n; ++i) {
            auto t = dsb::parse_trace(read_file(paths[i]));
            all.insert(all.end(), t.begin(), t.end());
        }
        std::stable_sort(all.begin(), all.end(), [](const dsb::Record& a, const dsb::Record& b) {
            return a.t != b.t ? a.t < b.t : a.seq < b.seq;
        });
        for (size_t i = 0; i < all.size(); ++i) all[i].seq = int64_t(i);
        write_file(out_path, dsb::trace_text(all));
        return DS_OK;
    });
}

ds_status ds_trace_report(const char* trace_path, int64_t n_stages, int64_t w0_us, int64_t w1_us,
                          uint64_t seed, char* report_json, size_t cap) {
    return guarded([&] {
        if (!trace_path || n_stages < 1) return ds_fail(DS_ERR_ARG, "bad trace report arguments");
        const auto tr = dsb::parse_trace(read_file(trace_path));
        copy_out(dsb::report_from_trace(tr, n_stages, w0_us, w1_us, seed).to_json(), report_json, cap, nullptr);
        return DS_OK;
    });
}

ds_status ds_report_kv(const char* report_json, const char* plan_json, int64_t latency_us,
                       const char* policy, char* out, size_t cap, size_t* needed) {
    return guarded([&] {
        if (!report_json || !plan_json) return ds_fail(DS_ERR_ARG, "null report/plan");
        const dsb::Report r = dsb::report_from_json(report_json);
        const dsb::Plan p = dsb::Plan::from_json(plan_json);
        copy_out(dsb::report_kv(r, p, latency_us, policy ? policy : ""), out, cap, needed);
        return DS_OK;
    });
}

ds_status ds_report_kv_priced(const char* report_json, const char* plan_json, int64_t latency_us,
                              const char* policy, const char* pricing_json, char* out, size_t cap,
                              size_t* needed) {
    return guarded([&] {
        if (!report_json || !plan_json || !pricing_json)
            return ds_fail(DS_ERR_ARG, "null report/plan/pricing");
        const dsb::Report r = dsb::report_from_json(report_json);
        const dsb::Plan p = dsb::Plan::from_json(plan_json);
        const dsb::Pricing pr = dsb::parse_pricing(pricing_json);
        copy_out(dsb::report_kv(r, p, latency_us, policy ? policy : "") +
                     dsb::profit_kv(dsb::analyze(r, pr)),
                 out, cap, needed);
        return DS_OK;
    });
}

ds_status ds_sweep_csv(const int64_t* lat, int32_t n_lat, const char* policies, const double* tput,
                       char* out, size_t cap, size_t* needed) {
    return guarded([&] {
        if (!lat || n_lat < 1 || !policies || !tput) return ds_fail(DS_ERR_ARG, "bad sweep arguments");
        std::vector<std::string> pol;
        std::stringstream ss(policies);
        std::string item;
        while (std::getline(ss, item, ',')) pol.push_back(item);
        const std::vector<int64_t> l(lat, lat + n_lat);
        const std::vector<double> v(tput, tput + pol.size() * size_t(n_lat));
        copy_out(dsb::sweep_csv(l, pol, v), out, cap, needed);
        return DS_OK;
    });
}

ds_status ds_session_limit(ds_session* h, int64_t max_circuits, int64_t* t0_us) {
    return guarded([&] {
        if (!h || !h->s) return ds_fail(DS_ERR_ARG, "null session");
        dsb::session_limit(h->s, max_circuits);
        if (t0_us) *t0_us = dsb::session_t0(h->s);
        return DS_OK;
    });
}

ds_status ds_session_capture(ds_session* h, const int64_t* reqs, int64_t n) {
    return guarded([&] {
        if (!h || !h->s || (n > 0 && !reqs)) return ds_fail(DS_ERR_ARG, "bad capture arguments");
        dsb::session_capture(h->s, std::vector<int64_t>(reqs, reqs + n));
        return DS_OK;
    });
}

ds_status ds_session_captured(ds_session* h, int64_t* meta4, float* logits, int64_t max_rows, int64_t* n_rows) {
    return guarded([&] {
        if (!h || !h->s) return ds_fail(DS_ERR_ARG, "null session");
        std::vector<int64_t> meta;
        const float* lg = nullptr;
        int64_t n = 0;
        dsb::session_captured(h->s, &meta, &lg, &n);
        if (n_rows) *n_rows = n;
        const int64_t k = std::min(n, max_rows);
        if (meta4 && k > 0) std::memcpy(meta4, meta.data(), size_t(k) * 4 * sizeof(int64_t));
        if (logits && k > 0) {
            const int64_t vocab = dsb::session_vocab(h->s);
            std::memcpy(logits, lg, size_t(k) * size_t(vocab) * 4);
        }
        return DS_OK;
    });
}

ds_status ds_run(const char* config_json, const char* config_dir, const char* policy, int64_t latency_us,
                 int64_t nb_override, const ds_model_desc* model, const ds_gpu_opts* opts,
                 const char* trace_path, char* report_json, size_t cap, size_t* needed) {
    return guarded([&] {
        if (!model || !opts) return ds_fail(DS_ERR_ARG, "null model/opts");
        ds_gpu_opts o = *opts;
        o.trace = 1;
        ds_session* h = nullptr;
        ds_status st = ds_session_create(config_json, config_dir, policy, latency_us, nb_override, model, &o, &h);
        if (st) return st;
        std::string js;
        try {
            dsb::GpuRunResult r = dsb::session_run(h->s, false, opts->collect_tokens != 0);
            if (!r.error.empty()) throw dsb::SimError(r.error);
            const auto tr = dsb::session_trace(h->s, -1, true);
            if (trace_path && *trace_path) write_file(trace_path, dsb::trace_text(tr));
            js = "{\"report\":" + trace_report_json(h->s, tr, -1, -1) + ",\"gpu\":" + r.to_json() + "}";
        } catch (...) {
            ds_session_destroy(h);
            throw;
        }
        ds_session_destroy(h);
        copy_out(js, report_json, cap, needed);
        return DS_OK;
    });
}

ds_status ds_session_destroy(ds_session* h) {
    return guarded([&] {
        if (h) dsb::session_destroy(h->s);
        delete h;
        return DS_OK;
    });
}

ds_status ds_gpu_run_config(const char* config_json, const char* config_dir, const char* policy,
                            int64_t latency_us, int64_t nb_override, const ds_model_desc* model,
                            const ds_gpu_opts* opts, char* report_json, size_t cap, size_t* needed) {
    return guarded([&] {
        if (!model || !opts) return ds_fail(DS_ERR_ARG, "null model/opts");
        auto cp = dsb::plan_from_config(config_json, config_dir, policy, latency_us, nb_override);
        dsb::SimOutput o = dsb::simulate(cp.second, cp.first.topo, cp.first.workload, cp.first.model,
                                         opts->trace != 0, true);
        dsb::GpuOptions g;
        g.device0 = opts->device0;
        g.n_devices = opts->n_devices;
        g.real_delay = opts->real_delay != 0;
        g.collect_tokens = opts->collect_tokens != 0;
        g.max_circuits = opts->max_circuits;
        g.weight_seed = opts->weight_seed;
        dsb::GpuRunResult r = dsb::run_on_gpus(cp.first, cp.second, o.schedule, *model, g);
        copy_out(r.to_json(), report_json, cap, needed);
        if (!r.error.empty()) return ds_fail(DS_ERR_RUNTIME, r.error);
        return DS_OK;
    });
}

}  // extern "C"
