// EventTrace text parsing and the SimReport recomputed from a trace. The GPU executor's
// real-clock traces carry the same integer fields as the virtual-clock schedule (replay mode,
// SURVEY.md 7.3 H7); their report must come from the trace itself, with the reference's
// definitions, so a hardware run and a virtual run are measured the same way.
#include <algorithm>
#include <cstdio>
#include <cstring>
#include <map>
#include <sstream>

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

}  // namespace dsb
