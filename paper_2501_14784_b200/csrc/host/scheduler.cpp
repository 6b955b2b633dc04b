// The microbatch scheduler of the stage-step path in virtual-clock mode: per-stage FIFO service,
// circuit composition (decode rows + a prefill chunk), the double-buffered KV swap plan, ring
// hops with latency + serialisation, admission/completion and the windowed report. Decision
// logic and tie-breaks restate the reference Engine (src/sim.cpp:95-587) so the trace is
// byte-identical; in addition every decision is recorded as a Schedule (circuits with their row
// layout, per-stage compute / swap / release ops) that the GPU executor replays verbatim
// (only timestamps differ on hardware).
#include <algorithm>
#include <deque>
#include <fstream>
#include <queue>
#include <sstream>

#include "pipeline.hpp"

namespace dsb {

const char* ev_name(Ev k) {
    switch (k) {
        case Ev::ComputeStart: return "ComputeStart";
        case Ev::ComputeEnd: return "ComputeEnd";
        case Ev::TransferArrive: return "TransferArrive";
        case Ev::SwapInDone: return "SwapInDone";
        case Ev::SwapOutDone: return "SwapOutDone";
        case Ev::RequestAdmit: return "RequestAdmit";
        case Ev::RequestComplete: return "RequestComplete";
    }
    return "?";
}

std::string trace_text(const std::vector<Record>& tr) {
    std::string out;
    out.reserve(tr.size() * 72);
    char buf[256];
    for (const Record& e : tr) {
        const int n = snprintf(buf, sizeof buf, "t=%lld seq=%lld kind=%s stage=%d mb=%d a=%lld b=%lld c=%lld\n",
                               (long long)e.t, (long long)e.seq, ev_name(e.kind), e.stage, e.mb,
                               (long long)e.a, (long long)e.b, (long long)e.c);
        out.append(buf, size_t(n));
    }
    return out;
}

std::string Report::to_json() const {
    std::ostringstream os;
    os.precision(17);
    os << "{\"window_start_us\":" << w0 << ",\"window_end_us\":" << w1 << ",\"input_tokens\":" << n_in
       << ",\"output_tokens\":" << n_out << ",\"wall_time_s\":" << wall_s
       << ",\"input_throughput\":" << in_tps << ",\"output_throughput\":" << out_tps
       << ",\"total_throughput\":" << total_tps << ",\"mean_bubble_fraction\":" << mean_bubble
       << ",\"max_bubble_fraction\":" << max_bubble << ",\"swap_stall_us\":" << swap_stall
       << ",\"completed_requests\":" << completed << ",\"live_requests\":" << live
       << ",\"admitted_requests\":" << admitted << ",\"rng_seed\":" << seed << ",\"stages\":[";
    for (size_t i = 0; i < stages.size(); ++i) {
        const auto& s = stages[i];
        os << (i ? "," : "") << "{\"busy_us\":" << s.busy << ",\"stall_us\":" << s.stall
           << ",\"bubble_us\":" << s.bubble << ",\"busy_fraction\":" << s.busy_frac
           << ",\"transfer_wait_fraction\":" << s.stall_frac << ",\"bubble_fraction\":" << s.bubble_frac
           << "}";
    }
    os << "]}";
    return os.str();
}

double analytic_throughput(const Plan& p) {
    const Micros circuit = p.S() * p.t_s + p.hop_latency_sum();
    const Micros period = std::max(p.n_mb * p.t_s, circuit);
    return double(p.n_mb * p.B()) * 1e6 / double(period);
}

std::pair<Tokens, Tokens> request_lengths(const Workload& w, int64_t k) {
    uint64_t st = w.seed + 0x9E3779B97F4A7C15ULL * uint64_t(k + 1);
    auto draw = [&st](Tokens lo, Tokens hi) {
        uint64_t z = (st += 0x9E3779B97F4A7C15ULL);
        z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ULL;
        z = (z ^ (z >> 27)) * 0x94D049BB133111EBULL;
        z ^= z >> 31;
        return lo + Tokens(z % (uint64_t(hi - lo) + 1));
    };
    const Tokens p = draw(w.prompt_min, w.prompt_max);
    const Tokens o = draw(w.output_min, w.output_max);
    return {p, o};
}

namespace {

// Request lengths: SplitMix64 keyed by (seed, index) (reference workload.cpp:11-53), or a
// fixed "prompt output" list that exhausts.
class Requests {
public:
    explicit Requests(const Workload& w) : w_(w) {
        if (w.trace_path.empty()) return;
        std::ifstream in(w.trace_path);
        if (!in) throw ConfigError("cannot open request trace " + w.trace_path);
        std::string line;
        while (std::getline(in, line)) {
            if (line.empty() || line[0] == '#') continue;
            std::replace(line.begin(), line.end(), ',', ' ');
            std::istringstream ls(line);
            Tokens p, o;
            if (!(ls >> p >> o)) throw ConfigError(w.trace_path + ": bad request line '" + line + "'");
            if (p < 0 || o < 0) throw ConfigError(w.trace_path + ": negative length in '" + line + "'");
            fixed_.emplace_back(p, o);
        }
    }
    std::pair<Tokens, Tokens> lengths(int64_t k) const {
        if (!fixed_.empty())
            return k < int64_t(fixed_.size()) ? fixed_[k] : std::pair<Tokens, Tokens>{-1, -1};
        return request_lengths(w_, k);
    }
    bool done() const { return !fixed_.empty() && next_ >= int64_t(fixed_.size()); }
    int64_t take() { return next_++; }

private:
    Workload w_;
    std::vector<std::pair<Tokens, Tokens>> fixed_;
    int64_t next_ = 0;
};

constexpr int rank_of(Ev k) {
    return k == Ev::ComputeEnd ? 0 : k == Ev::TransferArrive ? 1 : k == Ev::SwapInDone ? 2
                                 : k == Ev::SwapOutDone ? 3 : k == Ev::ComputeStart ? 4 : 5;
}

struct Pending {
    Micros t;
    int rank;
    int32_t stage, mb;
    int64_t order;
    Ev kind;
    int64_t a, b, c;
    bool operator>(const Pending& o) const {
        if (t != o.t) return t > o.t;
        if (rank != o.rank) return rank > o.rank;
        if (stage != o.stage) return stage > o.stage;
        if (mb != o.mb) return mb > o.mb;
        return order > o.order;
    }
};

enum class Residency : uint8_t { Absent, Loading, Resident };

struct Req {
    Tokens prompt = 0, target = 0, prompt_done = 0, generated = 0;
};

struct Mb {
    std::vector<int64_t> slot;  // request id or -1
    bool parked = true;
    int64_t eff = 0, n_decode = 0, live = 0;
    std::vector<std::pair<int64_t, Tokens>> prefill;  // (request, tokens) this circuit
    int64_t circuit = -1;
    int64_t trig = -1;  // circuit whose end sent this mb to stage 0 (Circuit::trig)
    Bytes trig_payload = 0;
};

struct StageRt {
    const Calibration* cal = nullptr;
    int64_t layers = 0;
    Bytes page = 0, local_cap = 0, m_global = 0, pcie = 0;
    const Link* out = nullptr;
    bool busy = false;
    Micros busy_since = 0;
    int64_t served = 0;
    std::deque<int32_t> queue;
    std::vector<Residency> res;
    std::vector<Micros> res_done;
    std::vector<Bytes> res_bytes;
    Bytes occupant[2] = {0, 0};
    Micros in_free = 0, out_free = 0;
    Micros busy_acc = 0, stall_acc = 0;
};

class VirtualPipeline {
public:
    VirtualPipeline(const Plan& p, const Topo& t, const Workload& w, const Model& m, bool trace,
                    bool sched)
        : plan_(p), topo_(t), wl_(w), model_(m), reqgen_(w), keep_trace_(trace), keep_sched_(sched) {}

    SimOutput run() {
        check();
        setup();
        Micros now = 0;
        while (!q_.empty()) {
            const Pending e = q_.top();
            if (e.t >= end_) break;
            q_.pop();
            now = e.t;
            switch (e.kind) {
                case Ev::ComputeStart: start_compute(e); break;
                case Ev::ComputeEnd: end_compute(e); break;
                case Ev::TransferArrive: {
                    StageRt& st = st_[e.stage];
                    st.queue.push_back(e.mb);
                    record(e.t, e.kind, e.stage, e.mb, e.a, e.b, 0);
                    dispatch(e.stage, e.t);
                    break;
                }
                case Ev::SwapInDone: {
                    StageRt& st = st_[e.stage];
                    if (st.res[e.mb] == Residency::Loading && st.res_done[e.mb] == e.t)
                        st.res[e.mb] = Residency::Resident;
                    record(e.t, e.kind, e.stage, e.mb, e.a, e.b, e.c);
                    dispatch(e.stage, e.t);
                    break;
                }
                case Ev::SwapOutDone: record(e.t, e.kind, e.stage, e.mb, e.a, e.b, e.c); break;
                default: throw SimError("unexpected queued event kind");
            }
        }
        if (q_.empty() && now < end_ && !admit_.empty()) {
            std::ostringstream os;
            os << "event-queue deadlock at t=" << now << "us: " << admit_.size()
               << " queued requests, microbatch states:";
            for (int32_t m = 0; m < NB_; ++m) os << " mb" << m << (mb_[m].parked ? "=parked" : "=active");
            throw SimError(os.str());
        }
        for (StageRt& st : st_)
            if (st.busy && st.busy_since < end_) st.busy_acc += overlap(st.busy_since, end_);
        SimOutput out;
        out.report = report();
        out.trace = std::move(trace_);
        out.schedule = std::move(sched_);
        return out;
    }

private:
    const Plan& plan_;
    const Topo& topo_;
    const Workload& wl_;
    const Model& model_;
    Requests reqgen_;
    bool keep_trace_, keep_sched_;

    int64_t S_ = 0, NB_ = 0, B_ = 0;
    bool swapping_ = false;
    Micros end_ = 0, w0_ = 0, w1_ = 0;
    std::vector<StageRt> st_;
    std::vector<Mb> mb_;
    std::vector<Req> req_;
    std::deque<int64_t> admit_;
    std::deque<int32_t> parked_;
    std::priority_queue<Pending, std::vector<Pending>, std::greater<Pending>> q_;
    int64_t order_ = 0;
    std::vector<Record> trace_;
    int64_t seq_ = 0;
    Schedule sched_;
    Tokens n_in_ = 0, n_out_ = 0;
    int64_t done_win_ = 0, done_all_ = 0, admitted_ = 0;

    void push(Micros t, Ev k, int32_t s, int32_t m, int64_t a = 0, int64_t b = 0, int64_t c = 0) {
        q_.push({t, rank_of(k), s, m, order_++, k, a, b, c});
    }
    void record(Micros t, Ev k, int32_t s, int32_t m, int64_t a = 0, int64_t b = 0, int64_t c = 0) {
        if (keep_trace_) trace_.push_back({t, seq_, k, s, m, a, b, c});
        ++seq_;
    }
    Micros overlap(Micros s, Micros e) const {
        const Micros lo = std::max(s, w0_), hi = std::min(e, w1_);
        return hi > lo ? hi - lo : 0;
    }
    bool in_win(Micros t) const { return t >= w0_ && t < w1_; }
    void op(int64_t s, OpKind k, int32_t m, int32_t slot, int64_t circ, int64_t bytes, Micros t) {
        if (keep_sched_) sched_.ops[s].push_back({k, m, slot, circ, bytes, t});
    }

    void check() const {
        if (plan_.stages.empty()) throw SimError("plan has no stages");
        if (plan_.n_mb < 1) throw SimError("plan has no microbatches");
        if (plan_.B() < 1) throw SimError("plan batch size must be >= 1");
        for (const auto& sp : plan_.stages)
            if (!topo_.node(sp.node_id))
                throw SimError("plan/topology mismatch: node " + sp.node_id + " not in topology");
        for (const auto& l : plan_.ring) {
            const Link* t = topo_.link(l.src, l.dst);
            if (!t || t->latency != l.latency || t->bw != l.bw)
                throw SimError("plan/topology mismatch: ring link " + l.src + "->" + l.dst +
                               " differs from topology");
        }
        const size_t want = plan_.stages.size() > 1 ? plan_.stages.size() : 0;
        if (plan_.ring.size() != want)
            throw SimError("plan/topology mismatch: expected " + std::to_string(want) +
                           " ring links, have " + std::to_string(plan_.ring.size()));
    }

    void new_request() {
        if (reqgen_.done()) return;
        const int64_t k = reqgen_.take();
        const auto [p, o] = reqgen_.lengths(k);
        if (p < 0) return;
        req_.push_back({p, o, 0, 0});
        admit_.push_back(k);
    }

    void setup() {
        S_ = plan_.S();
        NB_ = plan_.n_mb;
        B_ = plan_.B();
        swapping_ = plan_.offload && NB_ > 2;
        end_ = wl_.duration_s * 1'000'000;
        w0_ = wl_.warmup_s * 1'000'000;
        w1_ = end_;
        st_.resize(S_);
        if (keep_sched_) sched_.ops.assign(S_, {});
        for (int64_t i = 0; i < S_; ++i) {
            const StagePlanD& sp = plan_.stages[i];
            StageRt& st = st_[i];
            st.cal = &topo_.node(sp.node_id)->cal;
            st.layers = sp.layer_end - sp.layer_begin;
            st.page = page_size(model_, st.layers, model_.num_layers);
            st.m_global = sp.budget.m_global;
            st.local_cap = swapping_ ? sp.budget.local_bytes() : -1;
            st.pcie = sp.pcie;
            st.out = S_ > 1 ? &plan_.ring[i] : nullptr;
            st.res.assign(NB_, Residency::Absent);
            st.res_done.assign(NB_, 0);
            st.res_bytes.assign(NB_, 0);
        }
        mb_.resize(NB_);
        for (auto& m : mb_) m.slot.assign(B_, -1);
        for (int64_t i = 0; i < wl_.concurrency && !reqgen_.done(); ++i) {
            const int64_t k = reqgen_.take();
            const auto [p, o] = reqgen_.lengths(k);
            if (p < 0) break;
            req_.push_back({p, o, 0, 0});
            admit_.push_back(k);
        }
        for (int32_t m = 0; m < NB_; ++m) {
            fill(m, 0);
            if (mb_[m].live > 0) {
                mb_[m].parked = false;
                st_[0].queue.push_back(m);
                record(0, Ev::TransferArrive, 0, m, 0, 0);
            } else {
                parked_.push_back(m);
            }
        }
        dispatch(0, 0);
    }

    // admission into free slots, FIFO; zero-work requests finish on the spot (sim.cpp:244-275)
    void fill(int32_t m, Micros now) {
        Mb& mb = mb_[m];
        for (auto& slot : mb.slot) {
            if (slot != -1) continue;
            while (slot == -1 && !admit_.empty()) {
                const int64_t rid = admit_.front();
                admit_.pop_front();
                Req& r = req_[rid];
                ++admitted_;
                if (in_win(now)) n_in_ += r.prompt;
                record(now, Ev::RequestAdmit, -1, m, rid, r.prompt, r.target);
                if (r.prompt == 0 && r.target == 0) {
                    ++done_all_;
                    if (in_win(now)) ++done_win_;
                    record(now, Ev::RequestComplete, -1, m, rid, 0);
                    new_request();
                    continue;
                }
                slot = rid;
                ++mb.live;
            }
            if (admit_.empty() && slot == -1) break;
        }
    }

    void wake(Micros now, int64_t by_circuit) {
        while (!parked_.empty() && !admit_.empty()) {
            const int32_t m = parked_.front();
            fill(m, now);
            if (mb_[m].live == 0) break;
            parked_.pop_front();
            mb_[m].parked = false;
            const Bytes payload = mb_[m].live * plan_.policy.hidden_bytes_per_token;
            mb_[m].trig = by_circuit;
            mb_[m].trig_payload = payload;
            Micros hop = 0;
            if (S_ > 1) {
                const Link& l = plan_.ring.back();
                hop = l.latency + div_up(payload * 1'000'000, l.bw);
            }
            push(now + hop, Ev::TransferArrive, 0, m, now, payload);
        }
    }

    Bytes held_bytes(int32_t m, int64_t s) const {
        int64_t pages = 0;
        for (const int64_t rid : mb_[m].slot) {
            if (rid == -1) continue;
            const Tokens toks = req_[rid].prompt_done + req_[rid].generated;
            if (toks > 0) pages += div_up(toks, kPage);
        }
        return pages * st_[s].page;
    }

    Bytes offloaded_bytes(int32_t m, int64_t s) const {
        const StageRt& st = st_[s];
        if (st.local_cap < 0) return 0;
        const Bytes portion = held_bytes(m, s) - st.local_cap;
        if (portion <= 0) return 0;
        if (portion > st.m_global)
            throw SimError("microbatch KV exceeds local pool + global pool at stage " +
                           std::to_string(s) + " (admission sizing bug)");
        return portion;
    }

    int32_t next_live(int32_t m) const {
        for (int64_t k = 1; k <= NB_; ++k) {
            const int32_t c = int32_t((m + k) % NB_);
            if (!mb_[c].parked) return c;
        }
        return -1;
    }

    // evict the slot occupant (D2H), prefetch the target's offloaded portion (H2D) (sim.cpp:328-353)
    void prefetch(int64_t s, int32_t target, int slot, Micros now) {
        StageRt& st = st_[s];
        const Bytes out_b = st.occupant[slot];
        if (out_b > 0) {
            const Micros t0 = std::max(now, st.out_free);
            const Micros t1 = t0 + div_up(out_b * 1'000'000, st.pcie);
            st.out_free = t1;
            push(t1, Ev::SwapOutDone, int32_t(s), -1, t0, out_b, slot);
        }
        const Bytes in_b = offloaded_bytes(target, s);
        st.occupant[slot] = in_b;
        st.res_bytes[target] = in_b;
        op(s, OpKind::SwapIn, target, slot, -1, in_b, now);
        if (keep_sched_) sched_.ops[s].back().evict_bytes = out_b;
        if (in_b == 0) {
            st.res[target] = Residency::Resident;
            return;
        }
        const Micros t0 = std::max(now, st.in_free);
        const Micros t1 = t0 + div_up(in_b * 1'000'000, st.pcie);
        st.in_free = t1;
        st.res[target] = Residency::Loading;
        st.res_done[target] = t1;
        push(t1, Ev::SwapInDone, int32_t(s), target, t0, in_b, slot);
    }

    void dispatch(int64_t s, Micros now) {
        StageRt& st = st_[s];
        if (st.busy || st.queue.empty()) return;
        const int32_t m = st.queue.front();
        Micros start = now;
        if (swapping_) {
            if (st.res[m] == Residency::Absent) prefetch(s, m, int(st.served % 2), now);
            if (st.res[m] == Residency::Loading && st.res_done[m] > now) {
                st.stall_acc += overlap(now, st.res_done[m]);
                start = st.res_done[m];
            }
        }
        st.queue.pop_front();
        st.busy = true;
        if (s == 0) compose(m);
        push(start, Ev::ComputeStart, int32_t(s), m, mb_[m].eff, mb_[m].n_decode,
             swapping_ ? st.res_bytes[m] : 0);
    }

    // the circuit's rows: a prompt chunk shared over the slots in order, else one decode row
    // (sim.cpp:386-407); also the GPU row layout of this circuit at every stage
    void compose(int32_t m) {
        Mb& mb = mb_[m];
        mb.prefill.clear();
        mb.n_decode = 0;
        Tokens left = plan_.policy.prefill_chunk;
        Circuit c;
        c.mb = m;
        c.trig = mb.trig;
        c.trig_payload = mb.trig_payload;
        for (size_t si = 0; si < mb.slot.size(); ++si) {
            const int64_t rid = mb.slot[si];
            if (rid == -1) continue;
            const Req& r = req_[rid];
            if (r.prompt_done < r.prompt) {
                const Tokens take = std::min(left, r.prompt - r.prompt_done);
                if (take > 0) {
                    mb.prefill.emplace_back(rid, take);
                    left -= take;
                    const bool completes = r.prompt_done + take == r.prompt;
                    c.rows.push_back({int32_t(si), int32_t(r.prompt_done), int32_t(take),
                                      (completes && r.target > 0) ? 1 : 0, 0, rid});
                }
            } else {
                ++mb.n_decode;
                c.rows.push_back({int32_t(si), int32_t(r.prompt_done + r.generated), 1, 1, 1, rid});
            }
        }
        Tokens pre = 0;
        for (const auto& pr : mb.prefill) pre += pr.second;
        mb.eff = mb.n_decode + pre;
        if (keep_sched_) {
            c.eff_batch = mb.eff;
            c.n_decode = mb.n_decode;
            mb.circuit = int64_t(sched_.circuits.size());
            sched_.circuits.push_back(std::move(c));
        }
    }

    void start_compute(const Pending& e) {
        StageRt& st = st_[e.stage];
        st.busy_since = e.t;
        st.served++;
        record(e.t, e.kind, e.stage, e.mb, e.a, e.b, e.c);
        op(e.stage, OpKind::Compute, e.mb, -1, mb_[e.mb].circuit, e.c, e.t);
        if (swapping_) {
            st.res[e.mb] = Residency::Absent;
            const int32_t tgt = next_live(e.mb);
            if (tgt >= 0 && tgt != e.mb && st.res[tgt] == Residency::Absent)
                prefetch(e.stage, tgt, int(st.served % 2), e.t);
        }
        const Micros d = stage_time(*st.cal, std::max<int64_t>(1, e.a), st.layers,
                                    plan_.policy.calibration_ref_layers);
        push(e.t + d, Ev::ComputeEnd, e.stage, e.mb, e.a, e.b, e.stage == S_ - 1 ? 1 : 0);
    }

    void hop(int32_t m, int64_t from, Micros now) {
        const int64_t next = (from + 1) % S_;
        const Bytes payload = mb_[m].eff * plan_.policy.hidden_bytes_per_token;
        if (next == 0) {
            mb_[m].trig = mb_[m].circuit;
            mb_[m].trig_payload = payload;
        }
        Micros at = now;
        if (S_ > 1) {
            const Link& l = plan_.ring[from];
            at = now + l.latency + div_up(payload * 1'000'000, l.bw);
        }
        push(at, Ev::TransferArrive, int32_t(next), m, now, payload);
    }

    void end_compute(const Pending& e) {
        StageRt& st = st_[e.stage];
        st.busy = false;
        st.busy_acc += overlap(st.busy_since, e.t);
        record(e.t, e.kind, e.stage, e.mb, e.a, e.b, e.c);
        Mb& mb = mb_[e.mb];
        if (e.stage == S_ - 1) {
            Circuit* circ = keep_sched_ && mb.circuit >= 0 ? &sched_.circuits[mb.circuit] : nullptr;
            if (circ) circ->t_end = e.t;
            if (in_win(e.t)) n_out_ += mb.n_decode;
            for (const auto& [rid, take] : mb.prefill) req_[rid].prompt_done += take;
            for (size_t si = 0; si < mb.slot.size(); ++si) {
                int64_t& slot = mb.slot[si];
                if (slot == -1) continue;
                Req& r = req_[slot];
                bool prefilled_now = false;
                for (const auto& pr : mb.prefill)
                    if (pr.first == slot) prefilled_now = true;
                if (r.prompt_done == r.prompt && !prefilled_now) r.generated++;
                if (r.prompt_done == r.prompt && r.generated >= r.target) {
                    ++done_all_;
                    if (in_win(e.t)) ++done_win_;
                    record(e.t, Ev::RequestComplete, e.stage, e.mb, slot, r.generated);
                    if (circ) circ->completed_slots.push_back(int32_t(si));
                    for (int64_t s = 0; s < S_; ++s) op(s, OpKind::Release, e.mb, int32_t(si), -1, 0, e.t);
                    slot = -1;
                    --mb.live;
                    new_request();
                }
            }
            fill(e.mb, e.t);
            wake(e.t, mb.circuit);
            if (mb.live > 0) {
                hop(e.mb, e.stage, e.t);
            } else {
                mb.parked = true;
                parked_.push_back(e.mb);
            }
        } else {
            hop(e.mb, e.stage, e.t);
        }
        dispatch(e.stage, e.t);
    }

    Report report() const {
        Report r;
        r.w0 = w0_;
        r.w1 = w1_;
        r.n_in = n_in_;
        r.n_out = n_out_;
        const Micros win = w1_ - w0_;
        r.wall_s = double(win) / 1e6;
        r.in_tps = double(n_in_) * 1e6 / double(win);
        r.out_tps = double(n_out_) * 1e6 / double(win);
        r.total_tps = r.in_tps + r.out_tps;
        r.completed = done_win_;
        r.admitted = admitted_;
        r.live = admitted_ - done_all_;
        r.seed = wl_.seed;
        double sum = 0;
        for (const StageRt& st : st_) {
            StageStats s;
            s.busy = st.busy_acc;
            s.stall = st.stall_acc;
            s.bubble = win - st.busy_acc - st.stall_acc;
            s.busy_frac = double(s.busy) / double(win);
            s.stall_frac = double(s.stall) / double(win);
            s.bubble_frac = double(s.bubble) / double(win);
            r.max_bubble = std::max(r.max_bubble, s.bubble_frac);
            sum += s.bubble_frac;
            r.swap_stall += s.stall;
            r.stages.push_back(s);
        }
        r.mean_bubble = st_.empty() ? 0 : sum / double(S_);
        return r;
    }
};

}  // namespace

SimOutput simulate(const Plan& plan, const Topo& topo, const Workload& wl, const Model& model,
                   bool keep_trace, bool keep_schedule) {
    VirtualPipeline vp(plan, topo, wl, model, keep_trace, keep_schedule);
    return vp.run();
}

}  // namespace dsb
