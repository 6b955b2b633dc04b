// Perf model + planner: the integer sizing that fixes N_B, B, M_G and the KV pools the GPU
// stages allocate. Restates reference src/perf_model.cpp and src/planner.cpp; every result is
// checked bit-exact against the compiled reference (tests/test_integer_parity.py).
#include <algorithm>
#include <fstream>
#include <limits>
#include <set>
#include <sstream>

#include "json.hpp"
#include "pipeline.hpp"

namespace dsb {

const Node* Topo::node(const std::string& id) const {
    for (const auto& n : nodes)
        if (n.id == id) return &n;
    return nullptr;
}
const Link* Topo::link(const std::string& s, const std::string& d) const {
    for (const auto& l : links)
        if (l.src == s && l.dst == d) return &l;
    return nullptr;
}

// ------------------------------------------------------------------ calibration ----
// reference validate_calibration (perf_model.cpp:8-26)
void check_calibration(const Calibration& c) {
    if (c.size() < 2) throw std::runtime_error("calibration table needs at least two entries");
    for (size_t i = 0; i < c.size(); ++i) {
        if (c[i].batch < 1 || c[i].us <= 0)
            throw std::runtime_error("calibration entries must have batch >= 1 and time > 0");
        if (i && c[i].batch <= c[i - 1].batch)
            throw std::runtime_error("calibration batch sizes must strictly increase");
        if (i && c[i].us < c[i - 1].us)
            throw std::runtime_error("calibration times must be non-decreasing");
    }
}

// Paper Table 1 (reference perf_model.cpp:28-41)
const Calibration& table1() {
    static const Calibration t = {{1, 66600},  {2, 68900},  {4, 69100},   {8, 69500},  {16, 70300},
                                  {32, 76500}, {64, 80200}, {128, 89100}, {256, 137500}};
    return t;
}

// "batch,ms" rows, ms an exact decimal with <= 3 fractional digits (perf_model.cpp:44-83)
Calibration read_calibration_csv(const std::string& path) {
    std::ifstream in(path);
    if (!in) throw std::runtime_error("cannot open calibration file " + path);
    Calibration c;
    std::string line;
    while (std::getline(in, line)) {
        if (line.empty() || line[0] == '#') continue;
        const size_t comma = line.find(',');
        if (comma == std::string::npos) continue;
        std::string b = line.substr(0, comma), ms = line.substr(comma + 1);
        if (!b.empty() && !isdigit(static_cast<unsigned char>(b[0]))) continue;
        while (!ms.empty() && (ms.back() == '\r' || ms.back() == ' ')) ms.pop_back();
        const size_t dot = ms.find('.');
        std::string whole = dot == std::string::npos ? ms : ms.substr(0, dot);
        std::string frac = dot == std::string::npos ? "" : ms.substr(dot + 1);
        if (frac.size() > 3) throw std::runtime_error(path + ": sub-microsecond precision");
        frac.resize(3, '0');
        c.push_back({std::stoll(b), std::stoll(whole) * 1000 + std::stoll(frac)});
    }
    check_calibration(c);
    return c;
}

// piecewise-linear, half-up rounded; constant below, extrapolated above (perf_model.cpp:85-102)
Micros compute_time(const Calibration& c, int64_t batch) {
    check_calibration(c);
    if (batch < 1) throw std::runtime_error("batch_size must be >= 1");
    if (batch <= c.front().batch) return c.front().us;
    size_t seg = c.size() - 2;
    for (size_t k = 0; k + 1 < c.size(); ++k)
        if (batch <= c[k + 1].batch) {
            seg = k;
            break;
        }
    const CalPoint& lo = c[seg];
    const CalPoint& hi = c[seg + 1];
    if (batch == hi.batch) return hi.us;
    const int64_t span = hi.batch - lo.batch;
    const int64_t num = lo.us * span + (hi.us - lo.us) * (batch - lo.batch);
    return (num + span / 2) / span;
}

Micros stage_time(const Calibration& c, int64_t batch, int64_t layers, int64_t ref_layers) {
    const Micros t = compute_time(c, batch);
    if (ref_layers <= 0 || layers == ref_layers) return t;
    return mul_div_round(t, layers, ref_layers);
}

Bytes page_size(const Model& m, int64_t layers, int64_t total_layers) {
    if (layers <= 0 || total_layers <= 0 || layers > total_layers)
        throw std::invalid_argument("stage layer fraction must be in (0, 1]");
    return div_up(kPage * m.kv_bytes_per_token * layers, total_layers);
}

Bytes kv_size(const Model& m, Tokens tokens, int64_t layers, int64_t total_layers) {
    if (tokens < 0) throw std::invalid_argument("tokens must be >= 0");
    return tokens == 0 ? 0 : div_up(tokens, kPage) * page_size(m, layers, total_layers);
}

Bytes global_pool(Bytes pcie, Micros t, Bytes page) {
    if (pcie <= 0 || t <= 0 || page <= 0)
        throw std::invalid_argument("global_pool_size requires positive bandwidth, time, page");
    return pcie * t / 1'000'000 / page * page;
}

// Eq. 1 (perf_model.cpp:138-167)
Budget make_budget(const Node& n, Bytes weights, int64_t n_mb, Bytes m_global, bool offload) {
    if (n_mb < 1) throw PlanError("n_microbatches must be >= 1");
    Budget b;
    b.m_total = n.mem;
    b.m_weights = weights;
    b.m_kv = n.mem - weights;
    if (b.m_kv < 0)
        throw PlanError("weights-exceed-memory: node " + n.id + " needs " + std::to_string(weights) +
                        " weight bytes but has " + std::to_string(n.mem));
    b.n_mb = n_mb;
    b.offload = offload;
    b.m_global = offload ? m_global : 0;
    b.per_mb_plain = b.m_kv / n_mb;
    if (offload) {
        if (b.m_kv < 2 * b.m_global)
            throw PlanError("global-pools-exceed-kv-memory: node " + n.id + " has M_KV=" +
                            std::to_string(b.m_kv) + " < 2*M_G=" + std::to_string(2 * b.m_global));
        b.per_mb_offload = (b.m_kv - 2 * b.m_global) / n_mb + b.m_global;
    } else {
        b.per_mb_offload = b.per_mb_plain;
    }
    return b;
}

int64_t batch_fit(Bytes budget, const Model& m, int64_t layers, int64_t total_layers, Tokens seq) {
    if (seq < 1) throw std::invalid_argument("seq_len_budget must be >= 1");
    if (budget <= 0) return 0;
    return budget / kv_size(m, seq, layers, total_layers);
}

// ---------------------------------------------------------------------- planner ----
// largest-remainder proportional split of layers over usable memory (planner.cpp:19-78)
std::vector<std::pair<int64_t, int64_t>> split_layers(const Model& m, const Topo& t,
                                                      const std::vector<std::string>& order,
                                                      int64_t reserve_permille) {
    const int64_t L = m.num_layers;
    const int64_t n = int64_t(order.size());
    if (n < 1) throw PlanError("partition requires at least one node");
    if (n > L) throw PlanError("more nodes than layers");
    std::vector<Bytes> usable(n);
    Bytes usable_sum = 0, mem_sum = 0;
    for (int64_t i = 0; i < n; ++i) {
        const Node* nd = t.node(order[i]);
        if (!nd) throw PlanError("unknown node in ring order: " + order[i]);
        usable[i] = std::max<Bytes>(1, nd->mem - nd->mem * reserve_permille / 1000);
        usable_sum += usable[i];
        mem_sum += nd->mem;
    }
    if (mem_sum <= m.weight_bytes_total)
        throw PlanError("insufficient-total-memory: " + std::to_string(mem_sum) +
                        " bytes across nodes for " + std::to_string(m.weight_bytes_total) +
                        " weight bytes");
    std::vector<int64_t> cnt(n);
    std::vector<std::pair<Bytes, int64_t>> rem(n);
    int64_t given = 0;
    for (int64_t i = 0; i < n; ++i) {
        cnt[i] = L * usable[i] / usable_sum;
        rem[i] = {L * usable[i] % usable_sum, i};
        given += cnt[i];
    }
    std::sort(rem.begin(), rem.end(), [](const auto& a, const auto& b) {
        return a.first != b.first ? a.first > b.first : a.second < b.second;
    });
    for (int64_t k = 0; given < L; ++k, ++given) cnt[rem[k % n].second]++;
    for (int64_t i = 0; i < n; ++i)
        while (cnt[i] == 0) {
            auto mx = std::max_element(cnt.begin(), cnt.end());
            if (*mx <= 1) throw PlanError("cannot give every node a layer");
            --*mx;
            ++cnt[i];
        }
    std::vector<std::pair<int64_t, int64_t>> out(n);
    int64_t at = 0;
    for (int64_t i = 0; i < n; ++i) {
        out[i] = {at, at + cnt[i]};
        at += cnt[i];
    }
    return out;
}

int64_t bubble_free_nb(int64_t S, Micros t_s, Micros hop_sum) {
    if (t_s <= 0) throw PlanError("stage_time_us must be > 0");
    if (S < 1) throw PlanError("n_stages must be >= 1");
    return S + div_up(hop_sum, t_s);
}

std::vector<std::string> ring_order(const Topo& t, const std::string& mode) {
    std::vector<std::string> ids;
    for (const auto& n : t.nodes) ids.push_back(n.id);
    if (mode == "config" || ids.size() <= 2) return ids;
    if (mode != "nearest") throw PlanError("unknown ring_order mode: " + mode);
    std::vector<std::string> tour{ids.front()};
    std::vector<char> used(ids.size(), 0);
    used[0] = 1;
    while (tour.size() < ids.size()) {
        Micros best = -1;
        int64_t pick = -1;
        for (size_t i = 0; i < ids.size(); ++i) {
            if (used[i]) continue;
            const Link* l = t.link(tour.back(), ids[i]);
            const Micros lat = l ? l->latency : std::numeric_limits<Micros>::max();
            if (pick < 0 || lat < best) {
                best = lat;
                pick = int64_t(i);
            }
        }
        used[pick] = 1;
        tour.push_back(ids[pick]);
    }
    return tour;
}

static void check_topology(const Topo& t) {
    // first violation in canonical order decides the message (reference types.cpp:31-68)
    struct V { std::string kind, ent, msg; };
    std::vector<V> v;
    std::set<std::string> ids;
    for (const auto& n : t.nodes) {
        if (!ids.insert(n.id).second)
            v.push_back({"duplicate-node-id", n.id, "node_id '" + n.id + "' appears more than once"});
        if (n.mem <= 0) v.push_back({"nonpositive-gpu-mem", n.id, "gpu_mem_bytes must be > 0"});
        if (n.pcie <= 0)
            v.push_back({"nonpositive-pcie-bandwidth", n.id, "pcie_bandwidth_bytes_per_s must be > 0"});
    }
    for (const auto& l : t.links) {
        const std::string e = l.src + "->" + l.dst;
        if (l.src == l.dst) v.push_back({"self-loop", e, "link src and dst must differ"});
        if (!ids.count(l.src)) v.push_back({"unknown-endpoint", e, "link src '" + l.src + "' is not a node"});
        if (!ids.count(l.dst)) v.push_back({"unknown-endpoint", e, "link dst '" + l.dst + "' is not a node"});
        if (l.latency < 0) v.push_back({"negative-latency", e, "latency_us must be >= 0"});
        if (l.bw <= 0) v.push_back({"nonpositive-bandwidth", e, "bandwidth_bytes_per_s must be > 0"});
    }
    if (v.empty()) return;
    std::sort(v.begin(), v.end(), [](const V& a, const V& b) {
        if (a.kind != b.kind) return a.kind < b.kind;
        if (a.ent != b.ent) return a.ent < b.ent;
        return a.msg < b.msg;
    });
    throw PlanError("topology invalid: " + v.front().msg);
}

// fixed point batch -> T_S -> (N_B, M_G) -> budget -> batch, <= 32 rounds (planner.cpp:140-276)
Plan make_plan(const Model& m, const Topo& t, const Workload& w, const Policy& pol) {
    check_topology(t);
    const Tokens seq = w.prompt_max + w.output_max;
    if (seq < 1) throw PlanError("workload admits zero-size requests only");
    if (seq > m.max_seq_len)
        throw PlanError("per-request KV budget " + std::to_string(seq) +
                        " tokens exceeds model max_seq_len " + std::to_string(m.max_seq_len));
    const auto order = ring_order(t, pol.ring_order);
    const auto ranges = split_layers(m, t, order, pol.kv_reserve_permille);
    const int64_t S = int64_t(order.size());
    std::vector<Link> ring;
    if (S >= 2)
        for (int64_t i = 0; i < S; ++i) {
            const Link* l = t.link(order[i], order[(i + 1) % S]);
            if (!l)
                throw PlanError("missing-link: plan needs " + order[i] + " -> " + order[(i + 1) % S] +
                                " but the topology defines no such link");
            ring.push_back(*l);
        }
    Micros hop_sum = 0;
    for (const auto& l : ring) hop_sum += l.latency;

    struct Ctx {
        const Node* node;
        int64_t lb, le;
        Bytes weights, page, per_req;
    };
    std::vector<Ctx> cx(S);
    for (int64_t i = 0; i < S; ++i) {
        Ctx& c = cx[i];
        c.node = t.node(order[i]);
        c.lb = ranges[i].first;
        c.le = ranges[i].second;
        c.weights = m.layer_range_bytes(c.lb, c.le);
        if (i == 0) c.weights += m.embedding_bytes;
        if (i == S - 1) c.weights += m.output_layer_bytes;
        c.page = page_size(m, c.le - c.lb, m.num_layers);
        c.per_req = kv_size(m, seq, c.le - c.lb, m.num_layers);
        if (c.node->mem < c.weights)
            throw PlanError("weights-exceed-memory: node " + c.node->id + " cannot hold its stage weights");
    }
    int64_t batch = std::numeric_limits<int64_t>::max();
    for (const auto& c : cx)
        batch = std::min(batch, batch_fit((c.node->mem - c.weights) / S, m, c.le - c.lb, m.num_layers, seq));
    if (batch < 1) batch = 1;

    struct Iter {
        Micros t_s = 0;
        int64_t nb = 0, batch = 0;
        std::vector<Budget> budgets;
        std::vector<Micros> times;
    };
    Iter keep;
    bool converged = false;
    int64_t it = 1;
    for (; it <= 32; ++it) {
        Iter cur;
        cur.budgets.resize(S);
        cur.times.resize(S);
        for (int64_t i = 0; i < S; ++i) {
            cur.times[i] = stage_time(cx[i].node->cal, batch, cx[i].le - cx[i].lb, pol.calibration_ref_layers);
            cur.t_s = std::max(cur.t_s, cur.times[i]);
        }
        const Micros pool_t = pol.pool_time_basis == "slot" ? cur.t_s + hop_sum / S : cur.t_s;
        cur.nb = pol.nb_override > 0 ? pol.nb_override : bubble_free_nb(S, cur.t_s, hop_sum);
        int64_t next = std::numeric_limits<int64_t>::max();
        for (int64_t i = 0; i < S; ++i) {
            Bytes mg = 0;
            if (pol.offload) {
                mg = global_pool(cx[i].node->pcie, pool_t, cx[i].page);
                mg = mg * pol.pool_scale_milli / 1000 / cx[i].page * cx[i].page;
            }
            cur.budgets[i] = make_budget(*cx[i].node, cx[i].weights, cur.nb, mg, pol.offload);
            next = std::min(next, cur.budgets[i].per_mb() / cx[i].per_req);
        }
        if (next < 1) {
            if (keep.batch > 0) break;
            throw PlanError("infeasible-memory: not even one request per microbatch fits");
        }
        cur.batch = next;
        keep = std::move(cur);
        if (next == batch) {
            converged = true;
            break;
        }
        batch = next;
    }
    Plan p;
    p.n_mb = keep.nb;
    p.ring = ring;
    p.t_s = keep.t_s;
    p.offload = pol.offload;
    p.converged = converged;
    p.iterations = std::min<int64_t>(it, 32);
    p.seq_budget = seq;
    p.policy = pol;
    for (int64_t i = 0; i < S; ++i) {
        StagePlanD sp;
        sp.node_id = order[i];
        sp.layer_begin = cx[i].lb;
        sp.layer_end = cx[i].le;
        sp.weight_bytes = cx[i].weights;
        sp.pcie = cx[i].node->pcie;
        sp.budget = keep.budgets[i];
        sp.batch = keep.batch;
        sp.stage_time = keep.times[i];
        p.stages.push_back(sp);
    }
    return p;
}

// Same key order and formatting as the reference's nlohmann dump(2) (planner.cpp:294-335).
std::string Plan::to_json() const {
    using nlohmann::json;
    json j;
    j["n_microbatches"] = n_mb;
    j["stage_time_us"] = t_s;
    j["offload_enabled"] = offload;
    j["converged"] = converged;
    j["iterations"] = iterations;
    j["seq_budget_tokens"] = seq_budget;
    j["policy"] = {{"offload", policy.offload},
                   {"nb_override", policy.nb_override},
                   {"prefill_chunk", policy.prefill_chunk},
                   {"hidden_bytes_per_token", policy.hidden_bytes_per_token},
                   {"kv_reserve_permille", policy.kv_reserve_permille},
                   {"calibration_ref_layers", policy.calibration_ref_layers},
                   {"ring_order", policy.ring_order},
                   {"pool_scale_milli", policy.pool_scale_milli},
                   {"pool_time_basis", policy.pool_time_basis}};
    j["stages"] = json::array();
    for (const auto& s : stages)
        j["stages"].push_back({{"node_id", s.node_id},
                               {"layer_begin", s.layer_begin},
                               {"layer_end", s.layer_end},
                               {"stage_weight_bytes", s.weight_bytes},
                               {"pcie_bandwidth_bytes_per_s", s.pcie},
                               {"batch_size_per_microbatch", s.batch},
                               {"stage_time_us", s.stage_time},
                               {"budget",
                                {{"m_total", s.budget.m_total},
                                 {"m_weights", s.budget.m_weights},
                                 {"m_kv", s.budget.m_kv},
                                 {"m_global_pool", s.budget.m_global},
                                 {"n_microbatches", s.budget.n_mb},
                                 {"m_per_microbatch_no_offload", s.budget.per_mb_plain},
                                 {"m_per_microbatch_offload", s.budget.per_mb_offload},
                                 {"offload", s.budget.offload}}}});
    j["ring_links"] = json::array();
    for (const auto& l : ring)
        j["ring_links"].push_back({{"src", l.src},
                                   {"dst", l.dst},
                                   {"latency_us", l.latency},
                                   {"bandwidth_bytes_per_s", l.bw}});
    return j.dump(2) + "\n";
}

Plan Plan::from_json(const std::string& text) {
    using nlohmann::json;
    const json j = json::parse(text);
    Plan p;
    p.n_mb = j.at("n_microbatches").get<int64_t>();
    p.t_s = j.at("stage_time_us").get<Micros>();
    p.offload = j.at("offload_enabled").get<bool>();
    p.converged = j.at("converged").get<bool>();
    p.iterations = j.at("iterations").get<int64_t>();
    p.seq_budget = j.at("seq_budget_tokens").get<Tokens>();
    const json& pol = j.at("policy");
    p.policy.offload = pol.at("offload").get<bool>();
    p.policy.nb_override = pol.at("nb_override").get<int64_t>();
    p.policy.prefill_chunk = pol.at("prefill_chunk").get<int64_t>();
    p.policy.hidden_bytes_per_token = pol.at("hidden_bytes_per_token").get<Bytes>();
    p.policy.kv_reserve_permille = pol.at("kv_reserve_permille").get<int64_t>();
    p.policy.calibration_ref_layers = pol.at("calibration_ref_layers").get<int64_t>();
    p.policy.ring_order = pol.at("ring_order").get<std::string>();
    p.policy.pool_scale_milli = pol.at("pool_scale_milli").get<int64_t>();
    p.policy.pool_time_basis = pol.at("pool_time_basis").get<std::string>();
    for (const json& js : j.at("stages")) {
        StagePlanD s;
        s.node_id = js.at("node_id").get<std::string>();
        s.layer_begin = js.at("layer_begin").get<int64_t>();
        s.layer_end = js.at("layer_end").get<int64_t>();
        s.weight_bytes = js.at("stage_weight_bytes").get<Bytes>();
        s.pcie = js.at("pcie_bandwidth_bytes_per_s").get<Bytes>();
        s.batch = js.at("batch_size_per_microbatch").get<int64_t>();
        s.stage_time = js.at("stage_time_us").get<Micros>();
        const json& b = js.at("budget");
        s.budget.m_total = b.at("m_total").get<Bytes>();
        s.budget.m_weights = b.at("m_weights").get<Bytes>();
        s.budget.m_kv = b.at("m_kv").get<Bytes>();
        s.budget.m_global = b.at("m_global_pool").get<Bytes>();
        s.budget.n_mb = b.at("n_microbatches").get<int64_t>();
        s.budget.per_mb_plain = b.at("m_per_microbatch_no_offload").get<Bytes>();
        s.budget.per_mb_offload = b.at("m_per_microbatch_offload").get<Bytes>();
        s.budget.offload = b.at("offload").get<bool>();
        p.stages.push_back(s);
    }
    for (const json& l : j.at("ring_links"))
        p.ring.push_back({l.at("src").get<std::string>(), l.at("dst").get<std::string>(),
                          l.at("latency_us").get<Micros>(), l.at("bandwidth_bytes_per_s").get<Bytes>()});
    return p;
}

}  // namespace dsb
