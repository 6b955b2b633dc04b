// GPU executor: runs a plan's schedule on B200 stages in real time.
//
// The integer scheduler (scheduler.cpp) fixes, per stage, the ordered sequence of computes (with
// their circuit row layout), swap-ins and KV releases (SURVEY.md 7.3 H7 "replay mode"). Here one
// host thread per stage walks that sequence, launching the stage forward (ds_stage_step), the
// swap copies (ds_swap_in) and the hop to the next stage. Hops move activations [T, d] bf16
// device-to-device (peer copy when stages sit on different GPUs) and the sampled ids back to
// stage 0; the consumer may not start before producer completion + the injected link delay
// latency_us + ceil(payload * 1e6 / bw) (reference send_onward, src/sim.cpp:430-439), measured on
// the host clock from a stream callback at the producer's completion. Only timestamps differ from
// the virtual-clock trace; the integer contract (rows, swap bytes, slots) is executed verbatim.
#include <cuda_runtime.h>

#include <algorithm>
#include <atomic>
#include <chrono>
#include <condition_variable>
#include <cstring>
#include <memory>
#include <mutex>
#include <sstream>
#include <thread>

#include "capi_util.hpp"
#include "executor.hpp"
#include "pipeline.hpp"

namespace dsb {

std::pair<Config, Plan> plan_from_config(const char* json_text, const char* dir, const char* policy,
                                         int64_t latency_us, int64_t nb_override);

namespace {

int64_t now_us() {
    return std::chrono::duration_cast<std::chrono::microseconds>(
               std::chrono::steady_clock::now().time_since_epoch())
        .count();
}

#define XK(call)                                                                               \
    do {                                                                                       \
        cudaError_t e_ = (call);                                                               \
        if (e_ != cudaSuccess) throw SimError(std::string(#call) + ": " + cudaGetErrorString(e_)); \
    } while (0)
#define DK(call)                                                                         \
    do {                                                                                 \
        ds_status s_ = (call);                                                           \
        if (s_ != DS_OK) throw SimError(std::string(#call) + ": " + ds_last_error());    \
    } while (0)

struct Mailbox {
    std::mutex mu;
    std::condition_variable cv;
    int64_t posted = -1;  // circuit index delivered
    int64_t t_done = 0;   // host us when the producer's copy completed
    cudaEvent_t ev = nullptr;
};

struct PostCtx {
    Mailbox* box;
    int64_t circuit;
};

void CUDART_CB post_cb(void* p) {
    PostCtx* c = static_cast<PostCtx*>(p);
    {
        std::lock_guard<std::mutex> lk(c->box->mu);
        c->box->posted = c->circuit;
        c->box->t_done = now_us();
    }
    c->box->cv.notify_all();
    delete c;
}

struct StepTiming {
    cudaEvent_t a, b;
    int64_t rows;
};

struct Worker {
    int idx = 0;
    int device = 0;
    ds_stage* st = nullptr;
    cudaStream_t stream = nullptr;
    std::vector<std::unique_ptr<Mailbox>> in;  // per mb: input from the previous stage
    std::vector<void*> recv;                   // per mb: device buffer for that input
    std::vector<StepTiming> timing;
    int64_t served = 0, topups = 0;
    int64_t moved_in = 0, moved_out = 0, plan_in = 0;
    int64_t computes = 0;
    std::string error;
};

}  // namespace

GpuRunResult run_on_gpus(const Config& cfg, const Plan& plan, const Schedule& sched,
                         const ds_model_desc& md, const GpuOptions& opt) {
    const int64_t S = plan.S();
    const int64_t NB = plan.n_mb;
    int ndev = 0;
    if (cudaGetDeviceCount(&ndev) != cudaSuccess || ndev == 0)
        throw SimError("no CUDA device: the stage path has no CPU fallback");
    const int use_dev = opt.n_devices > 0 ? std::min(opt.n_devices, ndev) : ndev;
    const int64_t want_kv = int64_t(4) * md.n_kv_heads * md.d_head * md.n_layers;
    if (cfg.model.kv_bytes_per_token != want_kv)
        throw ConfigError("model kv_bytes_per_token " + std::to_string(cfg.model.kv_bytes_per_token) +
                          " != 4*n_kv*d_head*L = " + std::to_string(want_kv));

    // circuit limit and per-circuit bookkeeping
    const int64_t n_circ = opt.max_circuits > 0 ? std::min<int64_t>(opt.max_circuits, sched.circuits.size())
                                                : int64_t(sched.circuits.size());
    int64_t max_rows = 16, max_slot = 1;
    for (int64_t c = 0; c < n_circ; ++c) {
        max_rows = std::max(max_rows, sched.circuits[c].eff_batch);
        for (const auto& r : sched.circuits[c].rows) max_slot = std::max<int64_t>(max_slot, r.slot + 1);
    }
    max_rows = (max_rows + 15) / 16 * 16;
    const int64_t B = std::min<int64_t>(plan.B(), std::max<int64_t>(max_slot, 1));
    // previous circuit of the same microbatch (stage 0 input dependency)
    std::vector<int64_t> prev(n_circ, -1);
    {
        std::vector<int64_t> last(NB, -1);
        for (int64_t c = 0; c < n_circ; ++c) {
            prev[c] = last[sched.circuits[c].mb];
            last[sched.circuits[c].mb] = c;
        }
    }

    std::vector<Worker> W(S);
    const bool swapping = plan.offload && NB > 2;
    const Tokens ppr = div_up(plan.seq_budget, kPage);
    for (int64_t s = 0; s < S; ++s) {
        Worker& w = W[s];
        w.idx = int(s);
        w.device = opt.device0 + int(s % use_dev);
        const StagePlanD& sp = plan.stages[s];
        DK(ds_stage_create(w.device, &md, sp.layer_begin, sp.layer_end, s == 0, s == S - 1,
                           opt.weight_seed, int32_t(max_rows), int32_t(B), &w.st));
        const Bytes page = page_size(cfg.model, sp.layer_end - sp.layer_begin, cfg.model.num_layers);
        const Bytes need = B * ppr * page;  // a microbatch never holds more than this
        Bytes local = swapping ? sp.budget.local_bytes() : sp.budget.per_mb();
        local = std::min(local, need);
        const Bytes slot = swapping ? sp.budget.m_global : 0;
        DK(ds_kv_create(w.st, page, NB, local, slot, slot));
        void* sv = nullptr;
        DK(ds_stage_stream(w.st, &sv));
        w.stream = static_cast<cudaStream_t>(sv);
        XK(cudaSetDevice(w.device));
        w.in.resize(NB);
        w.recv.assign(NB, nullptr);
        for (int64_t m = 0; m < NB; ++m) {
            w.in[m].reset(new Mailbox());
            XK(cudaEventCreateWithFlags(&w.in[m]->ev, cudaEventDisableTiming));
            const size_t bytes = s == 0 ? size_t(max_rows) * 4 : size_t(max_rows) * md.d_model * 2;
            XK(cudaMalloc(&w.recv[m], bytes));
            XK(cudaMemset(w.recv[m], 0, bytes));
        }
    }
    if (use_dev > 1)
        for (int a = 0; a < use_dev; ++a)
            for (int b = 0; b < use_dev; ++b)
                if (a != b) {
                    int ok = 0;
                    cudaDeviceCanAccessPeer(&ok, opt.device0 + a, opt.device0 + b);
                    if (ok) {
                        cudaSetDevice(opt.device0 + a);
                        cudaDeviceEnablePeerAccess(opt.device0 + b, 0);
                        cudaGetLastError();
                    }
                }

    // sampled tokens (host, pinned) per circuit for the output streams
    std::vector<int32_t*> tok_host(n_circ, nullptr);
    int32_t* tok_pool = nullptr;
    std::vector<int64_t> tok_off(n_circ + 1, 0);
    for (int64_t c = 0; c < n_circ; ++c) {
        int64_t r = 0;
        for (const auto& row : sched.circuits[c].rows) r += row.need_logits;
        tok_off[c + 1] = tok_off[c] + r;
    }
    if (opt.collect_tokens && tok_off[n_circ] > 0) {
        XK(cudaMallocHost(&tok_pool, size_t(tok_off[n_circ]) * 4));
        for (int64_t c = 0; c < n_circ; ++c) tok_host[c] = tok_pool + tok_off[c];
    }

    auto hop_delay = [&](int64_t from, int64_t eff) -> int64_t {
        if (!opt.real_delay || S < 2) return 0;
        const Link& l = plan.ring[from];
        return l.latency + div_up(eff * plan.policy.hidden_bytes_per_token * 1'000'000, l.bw);
    };

    for (auto& w : W) {
        XK(cudaSetDevice(w.device));
        XK(cudaDeviceSynchronize());
    }
    std::atomic<bool> failed{false};
    const int64_t t0 = now_us();

    auto body = [&](Worker& w) {
        try {
            XK(cudaSetDevice(w.device));
            const int64_t s = w.idx;
            Worker& next = W[(s + 1) % S];
            std::vector<ds_row> rows;
            for (const StageOp& op : sched.ops[s]) {
                if (failed) return;
                if (op.kind == OpKind::Release) {
                    DK(ds_kv_release(w.st, op.mb, op.slot));
                    continue;
                }
                if (op.kind == OpKind::SwapIn) {
                    int64_t mi = 0, mo = 0;
                    DK(ds_swap_in(w.st, op.mb, op.slot, op.plan_bytes, &mi, &mo));
                    w.moved_in += mi;
                    w.moved_out += mo;
                    w.plan_in += op.plan_bytes;
                    continue;
                }
                const int64_t c = op.circuit;
                if (c < 0 || c >= n_circ) break;  // past the executed prefix
                const Circuit& circ = sched.circuits[c];
                const int32_t mb = circ.mb;
                w.served++;
                // ---- input dependency
                const int64_t need = s == 0 ? prev[c] : c;
                bool has_input = need >= 0;
                if (s == 0 && has_input) {
                    bool any_decode = false;
                    for (const auto& r : circ.rows) any_decode |= (r.is_decode && r.pos > 0);
                    has_input = any_decode;
                }
                if (has_input) {
                    Mailbox& mbx = *w.in[mb];
                    int64_t t_done;
                    {
                        std::unique_lock<std::mutex> lk(mbx.mu);
                        mbx.cv.wait(lk, [&] { return mbx.posted >= need || failed.load(); });
                        t_done = mbx.t_done;
                    }
                    if (failed) return;
                    const int64_t from = (s + S - 1) % S;
                    const int64_t arrive = t_done + hop_delay(from, sched.circuits[need].eff_batch);
                    const int64_t wait = arrive - now_us();
                    if (wait > 0) std::this_thread::sleep_for(std::chrono::microseconds(wait));
                    XK(cudaStreamWaitEvent(w.stream, mbx.ev, 0));
                }
                // ---- residency top-up: the plan's prefetch may be stale
                int32_t resident = 1;
                DK(ds_kv_resident(w.st, mb, &resident));
                if (!resident) {
                    int64_t mi = 0, mo = 0;
                    DK(ds_swap_in(w.st, mb, int32_t(w.served % 2), 0, &mi, &mo));
                    w.moved_in += mi;
                    w.moved_out += mo;
                    w.topups++;
                }
                // ---- the stage step
                rows.clear();
                for (const auto& r : circ.rows)
                    rows.push_back({r.slot, r.pos, r.n_tok, r.need_logits, r.is_decode, 0, r.req});
                StepTiming tm{};
                if (opt.step_timing) {
                    XK(cudaEventCreate(&tm.a));
                    XK(cudaEventCreate(&tm.b));
                    XK(cudaEventRecord(tm.a, w.stream));
                }
                const void* act_in = s == 0 ? (has_input ? w.recv[mb] : nullptr) : w.recv[mb];
                void* act_out = nullptr;
                const bool last = s == S - 1;
                if (last && S == 1) act_out = w.recv[mb];  // ids loop back to this stage
                DK(ds_stage_step(w.st, mb, rows.data(), int64_t(rows.size()), act_in, act_out));
                if (opt.step_timing) {
                    XK(cudaEventRecord(tm.b, w.stream));
                    tm.rows = circ.eff_batch;
                    w.timing.push_back(tm);
                }
                w.computes++;
                // ---- hop to the next stage (or ids back to stage 0)
                void* src = nullptr;
                int64_t bytes = 0, n_out = 0;
                DK(ds_stage_output(w.st, &src, &bytes, &n_out));
                if (last && S == 1) src = w.recv[mb];
                if (last && tok_host[c] && n_out > 0)
                    XK(cudaMemcpyAsync(tok_host[c], src, size_t(n_out) * 4, cudaMemcpyDeviceToHost, w.stream));
                if (S > 1 && bytes > 0) {
                    if (next.device == w.device)
                        XK(cudaMemcpyAsync(next.recv[mb], src, size_t(bytes), cudaMemcpyDeviceToDevice, w.stream));
                    else
                        XK(cudaMemcpyPeerAsync(next.recv[mb], next.device, src, w.device, size_t(bytes), w.stream));
                }
                Mailbox& out = *next.in[mb];
                XK(cudaEventRecord(out.ev, w.stream));
                XK(cudaLaunchHostFunc(w.stream, post_cb, new PostCtx{&out, c}));
            }
            XK(cudaStreamSynchronize(w.stream));
        } catch (const std::exception& e) {
            w.error = e.what();
            failed = true;
            for (auto& ww : W)
                for (auto& m : ww.in) m->cv.notify_all();
        }
    };
    std::vector<std::thread> th;
    for (auto& w : W) th.emplace_back(body, std::ref(w));
    for (auto& t : th) t.join();
    for (auto& w : W) {
        cudaSetDevice(w.device);
        ds_stage_sync(w.st);
    }
    const int64_t t1 = now_us();

    GpuRunResult res;
    for (auto& w : W)
        if (!w.error.empty() && res.error.empty()) res.error = "stage " + std::to_string(w.idx) + ": " + w.error;
    res.circuits = n_circ;
    res.wall_us = t1 - t0;
    for (int64_t c = 0; c < n_circ; ++c) {
        res.decode_tokens += sched.circuits[c].n_decode;
        res.rows += sched.circuits[c].eff_batch;
    }
    for (auto& w : W) {
        StageRunStats st;
        st.device = w.device;
        st.computes = w.computes;
        st.topups = w.topups;
        st.swap_plan_bytes = w.plan_in;
        st.swap_in_bytes = w.moved_in;
        st.swap_out_bytes = w.moved_out;
        for (auto& tm : w.timing) {
            float ms = 0;
            if (cudaEventElapsedTime(&ms, tm.a, tm.b) == cudaSuccess) {
                st.busy_ms += ms;
                st.steps.push_back({tm.rows, double(ms)});
            }
            cudaEventDestroy(tm.a);
            cudaEventDestroy(tm.b);
        }
        res.stages.push_back(std::move(st));
    }
    if (tok_pool) {
        res.tokens.resize(n_circ);
        for (int64_t c = 0; c < n_circ; ++c) res.tokens[c].assign(tok_host[c], tok_host[c] + (tok_off[c + 1] - tok_off[c]));
        cudaFreeHost(tok_pool);
    }
    for (auto& w : W) {
        cudaSetDevice(w.device);
        for (auto& m : w.in) cudaEventDestroy(m->ev);
        for (void* p : w.recv) cudaFree(p);
        ds_stage_destroy(w.st);
    }
    return res;
}

std::string GpuRunResult::to_json() const {
    std::ostringstream os;
    os.precision(10);
    os << "{\"circuits\":" << circuits << ",\"decode_tokens\":" << decode_tokens << ",\"rows\":" << rows
       << ",\"wall_us\":" << wall_us << ",\"tokens_per_s\":"
       << (wall_us > 0 ? double(decode_tokens) * 1e6 / double(wall_us) : 0.0) << ",\"error\":\"";
    for (char ch : error) os << (ch == '"' || ch == '\\' ? ' ' : ch);
    os << "\",\"stages\":[";
    for (size_t i = 0; i < stages.size(); ++i) {
        const auto& s = stages[i];
        os << (i ? "," : "") << "{\"device\":" << s.device << ",\"computes\":" << s.computes
           << ",\"busy_ms\":" << s.busy_ms << ",\"topups\":" << s.topups
           << ",\"swap_plan_bytes\":" << s.swap_plan_bytes << ",\"swap_in_bytes\":" << s.swap_in_bytes
           << ",\"swap_out_bytes\":" << s.swap_out_bytes << ",\"steps\":[";
        for (size_t k = 0; k < s.steps.size(); ++k)
            os << (k ? "," : "") << "[" << s.steps[k].first << "," << s.steps[k].second << "]";
        os << "]}";
    }
    os << "],\"tokens\":[";
    for (size_t c = 0; c < tokens.size(); ++c) {
        os << (c ? "," : "") << "[";
        for (size_t k = 0; k < tokens[c].size(); ++k) os << (k ? "," : "") << tokens[c][k];
        os << "]";
    }
    os << "]}";
    return os.str();
}

}  // namespace dsb
