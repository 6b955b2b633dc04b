// DeServe's profit model applied to hardware-run reports: the config's
// "pricing" section (reference src/config.cpp:58-70,169-199), the profitability analysis
// (src/economics.cpp:21-59) and the pricing block report_to_kv appends (src/sweep.cpp:187-194).
// Integer money (micro-dollars per hour, nano-dollars per token) and exact 128-bit products,
// so the block is byte-identical to the reference's for the same SimReport.
#include <cmath>
#include <cstdio>
#include <set>
#include <sstream>

#include "json.hpp"
#include "pipeline.hpp"

namespace dsb {

using nlohmann::json;

namespace {

// get_money (config.cpp:58-70): dollars -> integer units, rejecting finer than one unit.
int64_t money(const json& j, const std::string& key, int64_t unit_per_one) {
    if (!j.contains(key)) throw ConfigError("pricing: missing field '" + key + "'");
    const json& v = j.at(key);
    if (!v.is_number()) throw ConfigError("pricing." + key + ": expected a number");
    const double scaled = v.get<double>() * static_cast<double>(unit_per_one);
    const double rounded = std::llround(scaled);
    if (std::abs(scaled - rounded) > 1e-3)
        throw ConfigError("pricing." + key + ": finer than " + std::to_string(unit_per_one) +
                          " units per dollar");
    return static_cast<int64_t>(rounded);
}

// The bundled cost snapshots (economics.cpp:61-72): example data, not live rates.
const Pricing kPresets[] = {
    {"gcp-8xL4", 13'878'000, 900, 900, 900},
    {"runpod-8x4090", 5'520'000, 900, 900, 900},
    {"ionet-8x4090", 3'690'000, 900, 900, 900},
    {"whattomine-8x4090", 350'000, 900, 900, 900},
};

}  // namespace

Pricing parse_pricing(const std::string& text) {
    json j;
    try {
        j = json::parse(text);
    } catch (const json::parse_error& e) {
        throw ConfigError(std::string("pricing parse error: ") + e.what());
    }
    if (!j.is_object()) throw ConfigError("pricing: expected an object");
    auto only = [&](const std::set<std::string>& known) {
        for (auto it = j.begin(); it != j.end(); ++it)
            if (!known.count(it.key())) throw ConfigError("pricing: unknown field '" + it.key() + "'");
    };
    if (j.contains("preset")) {
        only({"preset"});
        if (!j.at("preset").is_string()) throw ConfigError("pricing.preset: expected a string");
        const std::string name = j.at("preset").get<std::string>();
        for (const Pricing& p : kPresets)
            if (p.name == name) return p;
        throw ConfigError("unknown pricing preset: " + name);
    }
    only({"compute_cost_per_hour", "price_per_token", "price_in_per_token", "price_out_per_token"});
    Pricing p;
    p.name = "config";
    p.cost_per_hour_micro = money(j, "compute_cost_per_hour", 1'000'000);
    if (j.contains("price_per_token")) p.price_nano = money(j, "price_per_token", 1'000'000'000);
    p.price_in_nano = j.contains("price_in_per_token") ? money(j, "price_in_per_token", 1'000'000'000)
                                                       : p.price_nano;
    p.price_out_nano = j.contains("price_out_per_token")
                           ? money(j, "price_out_per_token", 1'000'000'000)
                           : p.price_nano;
    if (p.price_nano == 0 && p.price_in_nano == 0 && p.price_out_nano == 0)
        throw ConfigError("pricing: no price fields given");
    return p;
}

Profit analyze(const Report& r, const Pricing& pr) {
    const Micros window = r.w1 - r.w0;
    if (window <= 0) throw SimError("analyze: report window is empty");
    if (r.n_in < 0 || r.n_out < 0) throw std::invalid_argument("token counts must be >= 0");
    if (pr.price_nano <= 0)
        throw std::invalid_argument("min_throughput requires a positive price per token");
    using i128 = __int128;
    Profit pa;
    // R = N_I * P_I + N_O * P_O in nano-dollars, floored to micro (economics.cpp:9-14)
    const i128 rev_nano = i128(r.n_in) * pr.price_in_nano + i128(r.n_out) * pr.price_out_nano;
    pa.revenue_micro = int64_t(rev_nano / 1000);
    // C * T: micro$/h * us / (3600e6 us/h)
    pa.cost_micro = int64_t(i128(pr.cost_per_hour_micro) * window / 3'600'000'000LL);
    pa.profit_micro = pa.revenue_micro - pa.cost_micro;
    // M_min = C / P tokens/s: (C micro$/h) / (P nano$/token) = 1000 C / P tokens/h
    pa.min_throughput = 1000.0 * double(pr.cost_per_hour_micro) / (3600.0 * double(pr.price_nano));
    pa.achieved_throughput = r.total_tps;
    // R > C*T on exact integers (nano$ * 3600e6 vs micro$ * 1000 * us)
    const i128 rhs = i128(pr.cost_per_hour_micro) * 1000 * window;
    const bool form1 = rev_nano * 3'600'000'000LL > rhs;
    if (pr.unified()) {  // M > C/P cross-multiplied: N * P * 36e8 > C * 1000 * T_us
        const bool form2 = i128(r.n_in + r.n_out) * pr.price_nano * 3'600'000'000LL > rhs;
        if (form1 != form2)
            throw SimError("profitability forms disagree (arithmetic bug): R>CT=" +
                           std::to_string(form1) + " M>C/P=" + std::to_string(form2));
    }
    pa.profitable = form1;
    return pa;
}

std::string profit_kv(const Profit& pa) {
    char buf[64];
    std::ostringstream os;
    os << "revenue_micro_usd=" << pa.revenue_micro << "\n"
       << "cost_micro_usd=" << pa.cost_micro << "\n"
       << "profit_micro_usd=" << pa.profit_micro << "\n";
    std::snprintf(buf, sizeof buf, "%.6f", pa.min_throughput);
    os << "min_throughput=" << buf << "\n";
    std::snprintf(buf, sizeof buf, "%.6f", pa.achieved_throughput);
    os << "achieved_throughput=" << buf << "\n"
       << "profitable=" << (pa.profitable ? 1 : 0) << "\n";
    return os.str();
}

}  // namespace dsb
