// EventTrace text parsing and the SimReport recomputed from a trace. The GPU executor's
// real-clock traces carry the same integer fields as the virtual-clock schedule (replay mode,
// SURVEY.md 7.3 H7); their report must come from the trace itself, with the reference's
// definitions, so a hardware run and a virtual run are measured the same way.
#include <algorithm>
#include <cstdio>
#include <cstring>
#include <map>
#include <sstream>

#include "json.hpp"
#include "pipeline.hpp"

namespace dsb {

namespace {
Ev ev_from_name(const std::string& n) {
    static const std::pair<const char*, Ev> k[] = {
        {"ComputeStart", Ev::ComputeStart}, {"ComputeEnd", Ev::ComputeEnd},
        {"TransferArrive", Ev::TransferArrive}, {"SwapInDone", Ev::SwapInDone},
        {"SwapOutDone", Ev::SwapOutDone}, {"RequestAdmit", Ev::RequestAdmit},
        {"RequestComplete", Ev::RequestComplete}};
    for (const auto& p : k)
        if (n == p.first) return p.second;
    throw ConfigError("trace: unknown event kind '" + n + "'");
}
}  // namespace

// Line format of reference write_trace (src/trace.cpp:40-46).
std::vector<Record> parse_trace(const std::string& text) {
    std::vector<Record> out;
    std::istringstream in(text);
    std::string line;
    while (std::getline(in, line)) {
        if (line.empty()) continue;
        long long t, seq, a, b, c;
        int stage, mb;
        char kind[32];
        if (sscanf(line.c_str(), "t=%lld seq=%lld kind=%31s stage=%d mb=%d a=%lld b=%lld c=%lld", &t, &seq,
                   kind, &stage, &mb, &a, &b, &c) != 8)
            throw ConfigError("trace: malformed line '" + line + "'");
        out.push_back({t, seq, ev_from_name(kind), stage, mb, a, b, c});
    }
    return out;
}

Report report_from_trace(const std::vector<Record>& tr, int64_t S, Micros w0, Micros w1, uint64_t seed) {
    if (w1 <= w0) throw SimError("report: empty window");
    auto overlap = [&](Micros s, Micros e) -> Micros {
        const Micros lo = std::max(s, w0), hi = std::min(e, w1);
        return hi > lo ? hi - lo : 0;
    };
    Report r;
    r.w0 = w0;
    r.w1 = w1;
    r.seed = seed;
    std::vector<Micros> busy(S, 0), stall(S, 0), since(S, -1), free_at(S, 0);
    std::map<std::pair<int32_t, int32_t>, Micros> arrived, swapped;
    int64_t done_all = 0;
    for (const Record& e : tr) {
        const bool in = e.t >= w0 && e.t < w1;
        const bool st_ok = e.stage >= 0 && e.stage < S;
        switch (e.kind) {
            case Ev::RequestAdmit:
                ++r.admitted;
                if (in) r.n_in += e.b;
                break;
            case Ev::RequestComplete:
                ++done_all;
                if (in) ++r.completed;
                break;
            case Ev::TransferArrive:
                if (st_ok) arrived[{e.stage, e.mb}] = e.t;
                break;
            case Ev::SwapInDone:
                if (st_ok) swapped[{e.stage, e.mb}] = e.t;
                break;
            case Ev::ComputeStart:
                if (!st_ok) break;
                since[e.stage] = e.t;
                if (e.c > 0) {  // waited for its global pages: engine stall_acc (sim.cpp:355-382)
                    auto a = arrived.find({e.stage, e.mb});
                    auto w = swapped.find({e.stage, e.mb});
                    const Micros ready = std::max(free_at[e.stage], a == arrived.end() ? 0 : a->second);
                    if (w != swapped.end() && w->second > ready)
                        stall[e.stage] += overlap(ready, std::min(w->second, e.t));
                }
                break;
            case Ev::ComputeEnd:
                if (!st_ok) break;
                if (since[e.stage] >= 0) busy[e.stage] += overlap(since[e.stage], e.t);
                since[e.stage] = -1;
                free_at[e.stage] = e.t;
                if (e.c == 1 && in) r.n_out += e.b;  // windowed_stats (workload.cpp:98-101)
                break;
            default:
                break;
        }
    }
    for (int64_t s = 0; s < S; ++s)
        if (since[s] >= 0) busy[s] += overlap(since[s], w1);  // still computing at the horizon
    r.live = r.admitted - done_all;
    const Micros win = w1 - w0;
    r.wall_s = double(win) / 1e6;
    r.in_tps = double(r.n_in) * 1e6 / double(win);
    r.out_tps = double(r.n_out) * 1e6 / double(win);
    r.total_tps = r.in_tps + r.out_tps;
    double sum = 0;
    for (int64_t s = 0; s < S; ++s) {
        StageStats x;
        x.busy = busy[s];
        x.stall = stall[s];
        x.bubble = win - busy[s] - stall[s];
        x.busy_frac = double(x.busy) / double(win);
        x.stall_frac = double(x.stall) / double(win);
        x.bubble_frac = double(x.bubble) / double(win);
        r.max_bubble = std::max(r.max_bubble, x.bubble_frac);
        sum += x.bubble_frac;
        r.swap_stall += x.stall;
        r.stages.push_back(x);
    }
    r.mean_bubble = S > 0 ? sum / double(S) : 0;
    return r;
}

Report report_from_json(const std::string& text) {
    const auto j = nlohmann::json::parse(text);
    Report r;
    r.w0 = j.at("window_start_us").get<int64_t>();
    r.w1 = j.at("window_end_us").get<int64_t>();
    r.n_in = j.at("input_tokens").get<int64_t>();
    r.n_out = j.at("output_tokens").get<int64_t>();
    r.wall_s = j.at("wall_time_s").get<double>();
    r.in_tps = j.at("input_throughput").get<double>();
    r.out_tps = j.at("output_throughput").get<double>();
    r.total_tps = j.at("total_throughput").get<double>();
    r.mean_bubble = j.at("mean_bubble_fraction").get<double>();
    r.max_bubble = j.at("max_bubble_fraction").get<double>();
    r.swap_stall = j.at("swap_stall_us").get<int64_t>();
    r.completed = j.at("completed_requests").get<int64_t>();
    r.live = j.at("live_requests").get<int64_t>();
    r.admitted = j.at("admitted_requests").get<int64_t>();
    r.seed = j.at("rng_seed").get<uint64_t>();
    for (const auto& s : j.at("stages")) {
        StageStats x;
        x.busy = s.at("busy_us").get<int64_t>();
        x.stall = s.at("stall_us").get<int64_t>();
        x.bubble = s.at("bubble_us").get<int64_t>();
        x.busy_frac = s.at("busy_fraction").get<double>();
        x.stall_frac = s.at("transfer_wait_fraction").get<double>();
        x.bubble_frac = s.at("bubble_fraction").get<double>();
        r.stages.push_back(x);
    }
    return r;
}

// The reference's key=value report (report_to_kv, src/sweep.cpp:146-195; no pricing block).
std::string report_kv(const Report& r, const Plan& p, Micros latency, const std::string& policy) {
    std::ostringstream os;
    char buf[64];
    auto f6 = [&](double v) {
        snprintf(buf, sizeof buf, "%.6f", v);
        return std::string(buf);
    };
    os << "seed=" << r.seed << "\n"
       << "policy=" << policy << "\n"
       << "latency_us=" << latency << "\n"
       << "n_stages=" << p.S() << "\n"
       << "n_microbatches=" << p.n_mb << "\n"
       << "batch_size=" << p.B() << "\n"
       << "stage_time_us=" << p.t_s << "\n"
       << "offload=" << (p.offload ? 1 : 0) << "\n"
       << "window_start_us=" << r.w0 << "\n"
       << "window_end_us=" << r.w1 << "\n"
       << "input_tokens=" << r.n_in << "\n"
       << "output_tokens=" << r.n_out << "\n"
       << "wall_time_s=" << f6(r.wall_s) << "\n"
       << "input_throughput=" << f6(r.in_tps) << "\n"
       << "output_throughput=" << f6(r.out_tps) << "\n"
       << "total_throughput=" << f6(r.total_tps) << "\n"
       << "mean_bubble_fraction=" << f6(r.mean_bubble) << "\n"
       << "max_bubble_fraction=" << f6(r.max_bubble) << "\n"
       << "swap_stall_us=" << r.swap_stall << "\n"
       << "completed_requests=" << r.completed << "\n"
       << "admitted_requests=" << r.admitted << "\n"
       << "live_requests=" << r.live << "\n";
    for (size_t i = 0; i < r.stages.size(); ++i) {
        const StageStats& s = r.stages[i];
        os << "stage." << i << ".busy_fraction=" << f6(s.busy_frac) << "\n"
           << "stage." << i << ".bubble_fraction=" << f6(s.bubble_frac) << "\n"
           << "stage." << i << ".transfer_wait_fraction=" << f6(s.stall_frac) << "\n"
           << "stage." << i << ".swap_stall_us=" << s.stall << "\n";
    }
    return os.str();
}

// The reference's sweep matrix (SweepResult::to_csv, src/sweep.cpp:68-82): a NaN cell = failed.
std::string sweep_csv(const std::vector<Micros>& lat, const std::vector<std::string>& pol,
                      const std::vector<double>& tput) {
    std::ostringstream os;
    os << "policy";
    for (Micros l : lat) os << "," << l;
    os << "\n";
    char buf[64];
    for (size_t i = 0; i < pol.size(); ++i) {
        os << pol[i];
        for (size_t k = 0; k < lat.size(); ++k) {
            const double v = tput[i * lat.size() + k];
            if (v != v) {
                os << ",failed";
            } else {
                snprintf(buf, sizeof buf, "%.3f", v);
                os << "," << buf;
            }
        }
        os << "\n";
    }
    return os.str();
}

}  // namespace dsb
