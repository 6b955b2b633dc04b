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
//
// A Session owns the stages (weights initialised once) so the schedule can be replayed many
// times (bench warm-up + timed runs); each run starts from empty KV pools.
#include <cuda_runtime.h>

#include <algorithm>
#include <atomic>
#include <chrono>
#include <condition_variable>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <memory>
#include <mutex>
#include <sstream>
#include <string>
#include <thread>

#include "capi_util.hpp"
#include "executor.hpp"
#include "hop_nccl.hpp"
#include "pipeline.hpp"

namespace dsb {

namespace {

const bool g_trace = getenv("DS_TRACE") != nullptr;

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

// stage 0 of a multi-stage pipeline: host time at which each circuit's output reached it (the
// last stage's completion in-process, the landing of its ids hop over NCCL); the arrival of a
// microbatch at stage 0 is timed from its trigger circuit (Circuit::trig)
struct CircuitDone {
    std::mutex mu;
    std::condition_variable cv;
    std::vector<int64_t> t;  // -1 until done
};

struct PostCtx {
    Mailbox* box;  // may be null
    int64_t circuit;
    CircuitDone* done = nullptr;
};

void CUDART_CB post_cb(void* p) {
    PostCtx* c = static_cast<PostCtx*>(p);
    const int64_t now = now_us();
    if (c->box) {
        {
            std::lock_guard<std::mutex> lk(c->box->mu);
            c->box->posted = std::max(c->box->posted, c->circuit);
            c->box->t_done = now;
        }
        c->box->cv.notify_all();
    }
    if (c->done) {
        {
            std::lock_guard<std::mutex> lk(c->done->mu);
            c->done->t[c->circuit] = now;
        }
        c->done->cv.notify_all();
    }
    if (g_trace) fprintf(stderr, "[ds] posted circuit %lld\n", (long long)c->circuit);
    delete c;
}

struct StepTiming {
    cudaEvent_t r = nullptr, a = nullptr, b = nullptr;  // ready, start (after swap wait), end
    int64_t rows = 0;
};

struct SwapTiming {
    cudaEvent_t e[4] = {nullptr, nullptr, nullptr, nullptr};  // in0, in1, out0, out1
};

struct Worker {
    int idx = 0;
    int device = 0;
    ds_stage* st = nullptr;
    cudaStream_t stream = nullptr;
    std::vector<std::unique_ptr<Mailbox>> in;  // per mb: input from the previous stage
    std::vector<void*> recv;                   // per mb: device buffer for that input
    std::vector<StepTiming> timing;            // event pool, reused across runs
    size_t timing_used = 0;
    cudaEvent_t t_begin = nullptr, t_end = nullptr;
    int64_t h_begin = 0;  // host steady-clock us at which t_begin fired (GPU -> host clock)
    int64_t served = 0, topups = 0;
    int64_t moved_in = 0, moved_out = 0, plan_in = 0;
    int64_t computes = 0;
    // per executed compute: host us of the microbatch's arrival and of its send (-1: derived
    // from the trigger's GPU end, single stage); per executed schedule swap-in: its events
    std::vector<int64_t> arr_us, send_us;
    std::vector<SwapTiming> swap_t;
    std::vector<SwapPair> swap_pairs;
    size_t swaps_done = 0;
    int phys_owner[2] = {-1, -1};  // microbatch physically holding each global slot
    int32_t last_mb = -1;          // microbatch of the latest enqueued compute (may still run)
    // per microbatch: op indices of its computes on this stage (slot choice looks ahead)
    std::vector<std::vector<int64_t>> comp_pos;
    std::string error;
    // per mb: the last circuit whose step (reading recv[mb]) is enqueued, and an event after it.
    // A producer may overwrite recv[mb] with the mb's next input only after that step: a circuit
    // without decode rows starts on stage 0 without waiting for its predecessor, so inputs of
    // one microbatch can otherwise overtake its unconsumed previous input.
    struct Sync {
        std::mutex mu;
        std::condition_variable cv;
    };
    std::unique_ptr<Sync> cs{new Sync()};
    std::vector<int64_t> consumed_c;
    std::vector<cudaEvent_t> consumed_ev;
};

}  // namespace

struct Session {
    Config cfg;
    Plan plan;
    Schedule sched;
    ds_model_desc md{};
    GpuOptions opt;
    int64_t n_circ = 0, max_rows = 16, B = 1;
    int64_t n_circ_all = 0;  // circuits prepared at creation; runs execute the first n_circ
    std::vector<int64_t> prev;
    std::vector<Worker> W;
    int32_t* tok_pool = nullptr;
    std::vector<int64_t> tok_off;
    // one-process-per-GPU mode: this process runs stage `rank`; hops go over NCCL
    bool nccl = false;
    int rank = 0, world = 1;
    const NcclApi* api = nullptr;
    RingLinks links;
    cudaStream_t s_send = nullptr, s_recv = nullptr;
    std::vector<void*> send_buf;        // ring of staged outputs for the sends
    std::vector<cudaEvent_t> ev_sent;   // per ring slot: its last send retired (slot reusable)
    int64_t send_seq = 0;
    int send_ring = 4;  // staging buffers: one per microbatch while they fit 1.5 GB (a slot
                        // reused while its send waits on the peer's receive couples the stages)
    std::vector<cudaEvent_t> ev_copy;   // per ring slot: output staged (send stream waits on it)
    std::vector<cudaEvent_t> ev_recv;   // per circuit: the receive of that circuit landed
    // receives in flight are bounded: a receive posted far ahead spins on the GPU and, once
    // NCCL's work queue fills, blocks the host inside ncclRecv while the peer waits on us
    static constexpr int kRecvAhead = 2;
    std::mutex land_mu;
    std::condition_variable land_cv;
    int64_t landed = 0;
    // NCCL mode, stage > 0: activation receives land in a ring of slots instead of one buffer
    // per microbatch (hundreds of microbatches with the opt policy at high latency). Slot k is
    // refilled once the step that read its previous occupant was enqueued (ev_consumed).
    bool ring_mode = false;
    std::vector<void*> recv_ring;
    std::vector<int32_t> recv_slot;        // per circuit
    std::vector<cudaEvent_t> ev_consumed;  // per slot
    std::vector<int64_t> consumed_n;       // per slot: consumptions enqueued (under land_mu)
    // real-clock trace
    std::vector<Record> vtrace;  // the virtual-clock trace of the schedule (opt.trace)
    CircuitDone done;
    int64_t t0 = 0, t_end = 0;   // host steady-clock us of the last run's start / end
    // logit capture
    std::vector<int64_t> cap_reqs;  // sorted
    std::vector<int64_t> cap_meta;  // 4 per row: circuit, req, position, row index
    float* cap_pool = nullptr;
    int64_t cap_rows = 0, cap_used = 0;
};

namespace {
struct LandCtx {
    Session* s;
};
void CUDART_CB land_cb(void* p) {
    Session* s = static_cast<LandCtx*>(p)->s;
    {
        std::lock_guard<std::mutex> lk(s->land_mu);
        s->landed++;
    }
    s->land_cv.notify_all();
    delete static_cast<LandCtx*>(p);
}
}  // namespace

Session* session_create(const Config& cfg, const Plan& plan, Schedule sched, const ds_model_desc& md,
                        const GpuOptions& opt, int rank, int world, const void* nccl_ids,
                        std::vector<Record> vtrace) {
    std::unique_ptr<Session> S(new Session());
    S->vtrace = std::move(vtrace);
    if (rank >= 0) {
        if (world != plan.S())
            throw ConfigError("world size " + std::to_string(world) + " != pipeline stages " +
                              std::to_string(plan.S()));
        S->nccl = world > 1;
        S->rank = rank;
        S->world = world;
    }
    S->cfg = cfg;
    S->plan = plan;
    S->sched = std::move(sched);
    S->md = md;
    S->opt = opt;
    const int64_t NS = plan.S();
    const int64_t NB = plan.n_mb;
    int ndev = 0;
    if (cudaGetDeviceCount(&ndev) != cudaSuccess || ndev == 0)
        throw SimError("no CUDA device: the stage path has no CPU fallback");
    const int use_dev = opt.n_devices > 0 ? std::min(opt.n_devices, ndev) : ndev;
    const int64_t want_kv = int64_t(4) * md.n_kv_heads * md.d_head * md.n_layers;
    if (cfg.model.kv_bytes_per_token != want_kv)
        throw ConfigError("model kv_bytes_per_token " + std::to_string(cfg.model.kv_bytes_per_token) +
                          " != 4*n_kv*d_head*L = " + std::to_string(want_kv));
    if (md.n_layers != cfg.model.num_layers) throw ConfigError("model layer count mismatch");

    const auto& circs = S->sched.circuits;
    S->n_circ = opt.max_circuits > 0 ? std::min<int64_t>(opt.max_circuits, circs.size())
                                     : int64_t(circs.size());
    int64_t max_slot = 1;
    for (int64_t c = 0; c < S->n_circ; ++c) {
        S->max_rows = std::max(S->max_rows, circs[c].eff_batch);
        for (const auto& r : circs[c].rows) max_slot = std::max<int64_t>(max_slot, r.slot + 1);
    }
    S->max_rows = (S->max_rows + 15) / 16 * 16;
    S->n_circ_all = S->n_circ;
    S->B = std::min<int64_t>(plan.B(), max_slot);
    S->prev.assign(S->n_circ, -1);
    {
        std::vector<int64_t> last(NB, -1);
        for (int64_t c = 0; c < S->n_circ; ++c) {
            S->prev[c] = last[circs[c].mb];
            last[circs[c].mb] = c;
        }
    }

    // in-process: every stage, stage s on device0 + s % n_devices; per-rank: only stage `rank`
    std::vector<int64_t> mine;
    if (rank >= 0)
        mine.push_back(rank);
    else
        for (int64_t s = 0; s < NS; ++s) mine.push_back(s);
    S->W.resize(mine.size());
    const bool swapping = plan.offload && NB > 2;
    const Tokens ppr = div_up(plan.seq_budget, kPage);
    for (size_t wi = 0; wi < mine.size(); ++wi) {
        const int64_t s = mine[wi];
        Worker& w = S->W[wi];
        w.idx = int(s);
        w.device = rank >= 0 ? opt.device0 : opt.device0 + int(s % use_dev);
        const StagePlanD& sp = plan.stages[s];
        DK(ds_stage_create(w.device, &md, sp.layer_begin, sp.layer_end, s == 0, s == NS - 1,
                           opt.weight_seed, int32_t(S->max_rows), int32_t(S->B), &w.st));
        const Bytes page = page_size(cfg.model, sp.layer_end - sp.layer_begin, cfg.model.num_layers);
        const Bytes need = S->B * ppr * page;  // a microbatch never holds more than this
        Bytes local = swapping ? sp.budget.local_bytes() : sp.budget.per_mb();
        local = std::min(local, need);
        const Bytes slot = swapping ? sp.budget.m_global : 0;
        DK(ds_kv_create(w.st, page, NB, local, slot, slot));
        void* sv = nullptr;
        DK(ds_stage_stream(w.st, &sv));
        w.stream = static_cast<cudaStream_t>(sv);
        XK(cudaSetDevice(w.device));
        XK(cudaEventCreate(&w.t_begin));
        XK(cudaEventCreate(&w.t_end));
        w.comp_pos.assign(NB, {});
        for (size_t oi = 0; oi < S->sched.ops[s].size(); ++oi)
            if (S->sched.ops[s][oi].kind == OpKind::Compute) w.comp_pos[S->sched.ops[s][oi].mb].push_back(int64_t(oi));
        w.in.resize(NB);
        w.recv.assign(NB, nullptr);
        w.consumed_c.assign(NB, -1);
        w.consumed_ev.assign(NB, nullptr);
        for (int64_t m = 0; m < NB; ++m)
            XK(cudaEventCreateWithFlags(&w.consumed_ev[m], cudaEventDisableTiming));
        // ring for activation receives when one buffer per microbatch would pass 1.5 GB
        const size_t slot_bytes = size_t(S->max_rows) * md.d_model * 2;
        // DS_RECV_RING=0 disables, =2 forces the ring (tests)
        const int ring_env = getenv("DS_RECV_RING") ? atoi(getenv("DS_RECV_RING")) : 1;
        const bool ring = S->nccl && s > 0 && ring_env != 0 &&
                          (ring_env == 2 || size_t(NB) * slot_bytes > (size_t(3) << 29));
        for (int64_t m = 0; m < NB; ++m) {
            w.in[m].reset(new Mailbox());
            if (ring) continue;
            const size_t bytes = s == 0 ? size_t(S->max_rows) * 4 : slot_bytes;
            XK(cudaMalloc(&w.recv[m], bytes));
            XK(cudaMemset(w.recv[m], 0, bytes));
        }
        if (ring) {
            // size: when this stage's compute needs receive j, all receives below the first
            // unconsumed index f are consumed, and posting j needs slot j % R free: R > j - f
            std::vector<int64_t> ridx(S->n_circ, -1);
            int64_t n_recv = 0;
            for (const StageOp& op : S->sched.ops[s - 1])
                if (op.kind == OpKind::Compute && op.circuit >= 0 && op.circuit < S->n_circ)
                    ridx[op.circuit] = n_recv++;
            std::vector<char> used(n_recv, 0);
            int64_t first = 0, need = 1;
            for (const StageOp& op : S->sched.ops[s])
                if (op.kind == OpKind::Compute && op.circuit >= 0 && op.circuit < S->n_circ &&
                    ridx[op.circuit] >= 0) {
                    const int64_t j = ridx[op.circuit];
                    need = std::max(need, j - first + 1);
                    used[j] = 1;
                    while (first < n_recv && used[first]) ++first;
                }
            const int64_t fit = int64_t((size_t(3) << 29) / slot_bytes);
            const int R = int(std::min<int64_t>(NB, std::max<int64_t>(need + Session::kRecvAhead + 1, fit)));
            S->ring_mode = true;
            S->recv_ring.assign(R, nullptr);
            S->ev_consumed.assign(R, nullptr);
            S->consumed_n.assign(R, 0);
            S->recv_slot.assign(S->n_circ, -1);
            for (int k = 0; k < R; ++k) {
                XK(cudaMalloc(&S->recv_ring[k], slot_bytes));
                XK(cudaMemset(S->recv_ring[k], 0, slot_bytes));
                XK(cudaEventCreateWithFlags(&S->ev_consumed[k], cudaEventDisableTiming));
            }
            w.recv[0] = S->recv_ring[0];  // warm-up target
        }
    }
    // a mailbox event is recorded on the PRODUCER's stream, so it must belong to that device
    for (auto& w : S->W) {
        const Worker& prod = S->nccl ? w : S->W[(w.idx + NS - 1) % NS];
        XK(cudaSetDevice(prod.device));
        for (auto& m : w.in) XK(cudaEventCreateWithFlags(&m->ev, cudaEventDisableTiming));
    }
    if (S->nccl) {
        std::string why;
        S->api = nccl_api(&why);
        if (!S->api) throw SimError("NCCL unavailable: " + why);
        Worker& w = S->W[0];
        XK(cudaSetDevice(w.device));
        XK(cudaStreamCreateWithFlags(&S->s_send, cudaStreamNonBlocking));
        XK(cudaStreamCreateWithFlags(&S->s_recv, cudaStreamNonBlocking));
        // a ring of staging buffers (one per microbatch unless 16 K-row prefill chunks would make
        // that gigabytes the planner budgeted for KV)
        const size_t sb = rank == NS - 1 ? size_t(S->max_rows) * 4 : size_t(S->max_rows) * md.d_model * 2;
        S->send_ring = int(std::max<int64_t>(4, std::min<int64_t>(NB, int64_t((size_t(3) << 29) / sb))));
        S->send_buf.assign(S->send_ring, nullptr);
        S->ev_copy.assign(S->send_ring, nullptr);
        S->ev_sent.assign(S->send_ring, nullptr);
        for (int k = 0; k < S->send_ring; ++k) {
            XK(cudaMalloc(&S->send_buf[k], sb));
            XK(cudaEventCreateWithFlags(&S->ev_copy[k], cudaEventDisableTiming));
            XK(cudaEventCreateWithFlags(&S->ev_sent[k], cudaEventDisableTiming));
        }
        S->ev_recv.assign(S->n_circ, nullptr);
        for (auto& e : S->ev_recv) XK(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
        S->links.init(*S->api, rank, world, static_cast<const ncclUniqueId*>(nccl_ids));
        // NCCL connects p2p peers lazily and the first send/recv on a link blocks the calling
        // host thread until the peer joins; warm both links up in one group so the send thread
        // and the receive thread never block on connection setup later
        S->links.warmup(*S->api, S->send_buf[0], w.recv[0], S->s_send);
        XK(cudaStreamSynchronize(S->s_send));
    }
    if (use_dev > 1 && rank < 0)
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
    S->done.t.assign(S->n_circ, -1);
    S->tok_off.assign(S->n_circ + 1, 0);
    for (int64_t c = 0; c < S->n_circ; ++c) {
        int64_t r = 0;
        for (const auto& row : circs[c].rows) r += row.need_logits;
        S->tok_off[c + 1] = S->tok_off[c] + r;
    }
    if (S->tok_off[S->n_circ] > 0) XK(cudaMallocHost(&S->tok_pool, size_t(S->tok_off[S->n_circ]) * 4));
    return S.release();
}

void session_destroy(Session* S) {
    if (!S) return;
    for (auto& w : S->W) {
        cudaSetDevice(w.device);
        cudaDeviceSynchronize();
        for (auto& m : w.in) cudaEventDestroy(m->ev);
        for (auto e : w.consumed_ev) cudaEventDestroy(e);
        if (!S->ring_mode)
            for (void* p : w.recv) cudaFree(p);
        for (void* p : S->recv_ring) cudaFree(p);
        for (auto e : S->ev_consumed) cudaEventDestroy(e);
        S->recv_ring.clear();
        S->ev_consumed.clear();
        for (auto& t : w.timing) {
            cudaEventDestroy(t.r);
            cudaEventDestroy(t.a);
            cudaEventDestroy(t.b);
        }
        if (w.t_begin) cudaEventDestroy(w.t_begin);
        if (w.t_end) cudaEventDestroy(w.t_end);
        ds_stage_destroy(w.st);
    }
    if (S->nccl) {
        for (void* p : S->send_buf) cudaFree(p);
        for (auto e : S->ev_copy) cudaEventDestroy(e);
        for (auto e : S->ev_sent) cudaEventDestroy(e);
        for (auto e : S->ev_recv) cudaEventDestroy(e);
        if (S->s_send) cudaStreamDestroy(S->s_send);
        if (S->s_recv) cudaStreamDestroy(S->s_recv);
        if (S->api) S->links.destroy(*S->api);
    }
    if (S->tok_pool) cudaFreeHost(S->tok_pool);
    if (S->cap_pool) cudaFreeHost(S->cap_pool);
    for (auto& w : S->W)
        for (auto& t : w.swap_t)
            for (auto e : t.e) cudaEventDestroy(e);
    delete S;
}

GpuRunResult session_run(Session* S, bool profile, bool collect_tokens) {
    const int64_t NS = S->plan.S();
    const auto& circs = S->sched.circuits;
    const Plan& plan = S->plan;
    const GpuOptions& opt = S->opt;
    for (auto& w : S->W) {
        XK(cudaSetDevice(w.device));
        DK(ds_kv_reset(w.st));
        DK(ds_stage_profile(w.st, profile ? 1 : 0));
        for (auto& m : w.in) m->posted = -1;
        S->landed = 0;
        w.served = w.topups = w.moved_in = w.moved_out = w.plan_in = w.computes = 0;
        std::fill(w.consumed_c.begin(), w.consumed_c.end(), int64_t(-1));
        std::fill(S->consumed_n.begin(), S->consumed_n.end(), 0);
        std::fill(S->recv_slot.begin(), S->recv_slot.end(), -1);
        w.timing_used = 0;
        w.arr_us.clear();
        w.send_us.clear();
        w.swap_pairs.clear();
        w.swaps_done = 0;
        w.phys_owner[0] = w.phys_owner[1] = -1;
        w.last_mb = -1;
        w.error.clear();
    }
    std::fill(S->done.t.begin(), S->done.t.end(), int64_t(-1));
    S->cap_used = 0;
    int64_t launches0 = 0;
    for (auto& w : S->W) {
        int64_t l = 0;
        DK(ds_stage_kernel_stats(w.st, nullptr, 0, &l));
        launches0 += l;
    }
    // bytes of the hop that lands at stage `to` for circuit c (activations, or ids at stage 0;
    // the ids hop always carries >= 1 int32 so stage 0 learns every circuit's end)
    auto hop_bytes = [&](int64_t to, int64_t c) -> size_t {
        if (to == 0) {
            int64_t r = 0;
            for (const auto& row : circs[c].rows) r += row.need_logits;
            return size_t(std::max<int64_t>(r, 1)) * 4;
        }
        return size_t(circs[c].eff_batch) * S->md.d_model * 2;
    };
    // injected delay of a hop carrying `payload` bytes over ring link `from` (send_onward /
    // wake_parked, sim.cpp:289,436)
    auto hop_delay = [&](int64_t from, int64_t payload) -> int64_t {
        if (!opt.real_delay || NS < 2) return 0;
        const Link& l = plan.ring[from];
        return l.latency + div_up(payload * 1'000'000, l.bw);
    };
    for (auto& w : S->W) {
        XK(cudaSetDevice(w.device));
        XK(cudaDeviceSynchronize());
        XK(cudaEventRecord(w.t_begin, w.stream));
        XK(cudaEventSynchronize(w.t_begin));
        w.h_begin = now_us();
    }
    std::atomic<bool> failed{false};
    const int64_t t0 = now_us();
    S->t0 = t0;
    // capture buffer: every sampled row of the captured requests in the executed prefix
    if (!S->cap_reqs.empty()) {
        int64_t n = 0;
        for (int64_t c = 0; c < S->n_circ; ++c)
            for (const auto& r : circs[c].rows)
                if (r.need_logits && std::binary_search(S->cap_reqs.begin(), S->cap_reqs.end(), r.req)) ++n;
        if (n > S->cap_rows) {
            if (S->cap_pool) cudaFreeHost(S->cap_pool);
            S->cap_pool = nullptr;
            XK(cudaMallocHost(&S->cap_pool, size_t(n) * S->md.vocab * 4));
            S->cap_rows = n;
        }
        S->cap_meta.clear();
    }

    // Physical global slot for a swap-in of `target` at op index `pos`: the plan's slot numbers
    // (served % 2, sim.cpp:417-421) are its integer contract and stay in the trace, but the
    // plan does not mark a microbatch absent when another prefetch reuses its slot (SURVEY.md
    // H3), so following them evicts microbatches just before they compute. The executor knows
    // the whole op sequence: it keeps the target where it already is, else uses an empty slot,
    // else never evicts the microbatch of the latest launched compute (its refill would wait for
    // that step to finish and then stall the next one), else evicts the occupant whose next
    // compute comes later. DS_SWAP_SLOTS=plan: the plan's numbers; =lookahead: no pinning.
    // Measured with the early top-up (profiles/r02_swap_slot_policies.md): 70B 4-stage swap
    // 582.8 tok/s pinned vs 521.2 lookahead, 8B 4-stage swap 3,042 vs 3,013; pinning doubles the
    // top-ups, which the early top-up overlaps with the hop.
    static const std::string slot_env = getenv("DS_SWAP_SLOTS") ? getenv("DS_SWAP_SLOTS") : "";
    static const bool plan_slots = slot_env == "plan";
    static const bool pin_last = slot_env != "lookahead";
    auto pick_slot = [&](Worker& w, int32_t target, int64_t pos, int plan_slot) -> int {
        if (plan_slots) return plan_slot;
        for (int k = 0; k < 2; ++k)
            if (w.phys_owner[k] == target) return k;
        for (int k : {plan_slot, 1 - plan_slot})
            if (w.phys_owner[k] < 0) return k;
        if (pin_last)
            for (int k = 0; k < 2; ++k)
                if (w.phys_owner[k] == w.last_mb) return 1 - k;
        auto next_use = [&](int32_t m) -> int64_t {
            const auto& v = w.comp_pos[m];
            auto it = std::upper_bound(v.begin(), v.end(), pos);
            return it == v.end() ? INT64_MAX : *it;
        };
        const int64_t u0 = next_use(w.phys_owner[0]), u1 = next_use(w.phys_owner[1]);
        if (u0 == u1) return plan_slot;
        return u0 > u1 ? 0 : 1;
    };
    auto note_swap = [](Worker& w, int32_t target, int slot) {
        if (w.phys_owner[1 - slot] == target) w.phys_owner[1 - slot] = -1;
        w.phys_owner[slot] = target;
    };

    auto body = [&](Worker& w) {
        try {
            XK(cudaSetDevice(w.device));
            const int64_t s = w.idx;
            Worker* next = S->nccl ? nullptr : &S->W[(s + 1) % NS];
            const bool last = s == NS - 1;
            std::vector<ds_row> rows;
            const auto& ops = S->sched.ops[s];
            for (size_t oi = 0; oi < ops.size(); ++oi) {
                const StageOp& op = ops[oi];
                if (failed) return;
                if (op.kind == OpKind::Release) {
                    DK(ds_kv_release(w.st, op.mb, op.slot));
                    continue;
                }
                if (op.kind == OpKind::SwapIn) {
                    if (w.swaps_done == w.swap_t.size()) {
                        SwapTiming t;
                        for (auto& e : t.e) XK(cudaEventCreate(&e));
                        w.swap_t.push_back(t);
                    }
                    SwapTiming& t = w.swap_t[w.swaps_done++];
                    DK(ds_swap_events(w.st, t.e[0], t.e[1], t.e[2], t.e[3]));
                    int64_t mi = 0, mo = 0;
                    const int ps = pick_slot(w, op.mb, int64_t(oi), op.slot);
                    DK(ds_swap_in(w.st, op.mb, ps, op.plan_bytes, &mi, &mo));
                    note_swap(w, op.mb, ps);
                    w.moved_in += mi;
                    w.moved_out += mo;
                    w.plan_in += op.plan_bytes;
                    int64_t sw[4] = {0, 0, 0, 0};
                    DK(ds_swap_stats(w.st, sw));
                    w.swap_pairs.push_back({op.plan_bytes, sw[0], sw[1], sw[2]});
                    continue;
                }
                const int64_t c = op.circuit;
                if (c < 0 || c >= S->n_circ) break;  // past the executed prefix
                const Circuit& circ = circs[c];
                const int32_t mb = circ.mb;
                w.served++;
                // ---- residency top-up: the plan's prefetch may be stale, or the
                // step's growth may exceed the whole local pages before the plan's byte figure
                // shows a global portion. Checked before the input wait, so the refill copy
                // overlaps the hop (and the previous step) instead of delaying this step; the
                // copies still wait for the evicted occupant's last compute and the step waits
                // for the refill.
                rows.clear();
                for (const auto& r : circ.rows)
                    rows.push_back({r.slot, r.pos, r.n_tok, r.need_logits, r.is_decode, 0, r.req});
                int32_t resident = 1;
                DK(ds_kv_ready(w.st, mb, rows.data(), int64_t(rows.size()), &resident));
                if (!resident) {
                    int64_t mi = 0, mo = 0;
                    DK(ds_swap_events(w.st, nullptr, nullptr, nullptr, nullptr));
                    const int ps = pick_slot(w, mb, int64_t(oi), int(w.served % 2));
                    DK(ds_swap_in(w.st, mb, ps, 0, &mi, &mo));
                    note_swap(w, mb, ps);
                    w.moved_in += mi;
                    w.moved_out += mo;
                    w.topups++;
                }
                // ---- input dependency: previous stage, or (stage 0) this mb's previous circuit
                const int64_t need = s == 0 ? S->prev[c] : c;
                bool has_input = need >= 0;
                if (s == 0 && has_input) {
                    bool any_decode = false;
                    for (const auto& r : circ.rows) any_decode |= (r.is_decode && r.pos > 0);
                    has_input = any_decode;
                }
                int64_t arr = -1, sent = -1;  // trace: arrival / send time (host us)
                if (s == 0 && NS > 1) {
                    // the microbatch arrives from the last stage: send_onward of its previous
                    // circuit, or wake_parked by another microbatch's circuit end (Circuit::trig)
                    if (circ.trig >= 0) {
                        if (has_input && circ.trig != need)
                            throw SimError("circuit " + std::to_string(c) + " has decode rows but was woken");
                        {
                            std::unique_lock<std::mutex> lk(S->done.mu);
                            S->done.cv.wait(lk, [&] { return S->done.t[circ.trig] >= 0 || failed.load(); });
                            sent = S->done.t[circ.trig];
                        }
                        if (failed) return;
                        const int64_t arrive = sent + hop_delay(NS - 1, circ.trig_payload);
                        const int64_t wait = arrive - now_us();
                        if (wait > 0) std::this_thread::sleep_for(std::chrono::microseconds(wait));
                        arr = std::max(arrive, now_us());
                        if (has_input)
                            XK(cudaStreamWaitEvent(w.stream, S->nccl ? S->ev_recv[need] : w.in[mb]->ev, 0));
                    } else {
                        arr = sent = t0;  // placed at t = 0
                    }
                } else if (s > 0) {
                    // single stage: the input is this stream's own previous step (ids loop back
                    // on the device, no link, no injected delay: reference sim.cpp:434-437), so
                    // stream order is the dependency and the host runs ahead of the GPU
                    Mailbox& mbx = *w.in[mb];
                    int64_t t_done;
                    {
                        std::unique_lock<std::mutex> lk(mbx.mu);
                        if (g_trace) fprintf(stderr, "[ds r%lld] wait c=%lld mb=%d need=%lld posted=%lld\n", (long long)s, (long long)c, mb, (long long)need, (long long)mbx.posted);
                        mbx.cv.wait(lk, [&] { return mbx.posted >= need || failed.load(); });
                        t_done = mbx.t_done;
                    }
                    if (failed) return;
                    const int64_t from = (s + NS - 1) % NS;
                    const int64_t arrive =
                        t_done + hop_delay(from, circs[need].eff_batch * plan.policy.hidden_bytes_per_token);
                    const int64_t wait = arrive - now_us();
                    if (wait > 0) std::this_thread::sleep_for(std::chrono::microseconds(wait));
                    arr = std::max(arrive, now_us());
                    sent = t_done;
                    XK(cudaStreamWaitEvent(w.stream, S->nccl ? S->ev_recv[need] : mbx.ev, 0));
                }
                w.arr_us.push_back(arr);
                w.send_us.push_back(sent);
                // ---- the stage step
                StepTiming* tm = nullptr;
                if (opt.step_timing) {
                    if (w.timing_used == w.timing.size()) {
                        StepTiming n;
                        XK(cudaEventCreate(&n.r));
                        XK(cudaEventCreate(&n.a));
                        XK(cudaEventCreate(&n.b));
                        w.timing.push_back(n);
                    }
                    tm = &w.timing[w.timing_used++];
                    tm->rows = circ.eff_batch;
                    DK(ds_stage_step_events(w.st, tm->r, tm->a, tm->b));
                }
                int32_t ring_slot = -1;
                if (S->ring_mode && s > 0) ring_slot = S->recv_slot[c];
                const void* act_in = s == 0 ? (has_input ? w.recv[mb] : nullptr)
                                            : (ring_slot >= 0 ? S->recv_ring[ring_slot] : w.recv[mb]);
                void* act_out = (last && NS == 1) ? w.recv[mb] : nullptr;  // ids loop back
                DK(ds_stage_step(w.st, mb, rows.data(), int64_t(rows.size()), act_in, act_out));
                w.last_mb = mb;
                XK(cudaEventRecord(w.consumed_ev[mb], w.stream));  // recv[mb] read by this step
                if (ring_slot >= 0) {  // the ring slot may be refilled once this step has read it
                    XK(cudaEventRecord(S->ev_consumed[ring_slot], w.stream));
                    {
                        std::lock_guard<std::mutex> lk(S->land_mu);
                        S->consumed_n[ring_slot]++;
                    }
                    S->land_cv.notify_all();
                }
                {
                    std::lock_guard<std::mutex> lk(w.cs->mu);
                    w.consumed_c[mb] = c;
                }
                w.cs->cv.notify_all();
                if (g_trace) fprintf(stderr, "[ds r%lld] step c=%lld mb=%d rows=%lld need=%lld\n", (long long)s, (long long)c, mb, (long long)circ.eff_batch, (long long)need);
                w.computes++;
                // logits of captured requests (teacher-forced parity, tests)
                if (last && !S->cap_reqs.empty()) {
                    const float* lg = nullptr;
                    int64_t lr = 0, k = 0;
                    DK(ds_stage_logits_device(w.st, &lg, &lr));
                    for (const auto& r : circ.rows) {
                        if (!r.need_logits) continue;
                        if (std::binary_search(S->cap_reqs.begin(), S->cap_reqs.end(), r.req)) {
                            if (S->cap_used >= S->cap_rows) throw SimError("logit capture overflow");
                            const size_t V = size_t(S->md.vocab);
                            XK(cudaMemcpyAsync(S->cap_pool + size_t(S->cap_used) * V, lg + size_t(k) * V,
                                               V * 4, cudaMemcpyDeviceToHost, w.stream));
                            S->cap_meta.insert(S->cap_meta.end(), {c, r.req, int64_t(r.pos + r.n_tok - 1), k});
                            S->cap_used++;
                        }
                        ++k;
                    }
                }
                // ---- hop to the next stage (or ids back to stage 0)
                void* src = nullptr;
                int64_t bytes = 0, n_out = 0;
                DK(ds_stage_output(w.st, &src, &bytes, &n_out));
                if (last && NS == 1) src = w.recv[mb];
                if (last && collect_tokens && S->tok_pool && n_out > 0)
                    XK(cudaMemcpyAsync(S->tok_pool + S->tok_off[c], src, size_t(n_out) * 4,
                                       cudaMemcpyDeviceToHost, w.stream));
                if (S->nccl) {
                    // stage the output per microbatch, then ncclSend on the send stream (the ids
                    // hop carries at least one int32: stage 0 times every circuit end)
                    if (last && bytes == 0) bytes = 4;
                    if (bytes > 0) {
                        const int k = int(S->send_seq++ % S->send_ring);
                        XK(cudaStreamWaitEvent(w.stream, S->ev_sent[k], 0));  // slot's last send done
                        XK(cudaMemcpyAsync(S->send_buf[k], src, size_t(bytes), cudaMemcpyDeviceToDevice,
                                           w.stream));
                        XK(cudaEventRecord(S->ev_copy[k], w.stream));
                        XK(cudaStreamWaitEvent(S->s_send, S->ev_copy[k], 0));
                        const ncclResult_t nr = S->api->Send(S->send_buf[k], size_t(bytes), ncclUint8, 1,
                                                             S->links.send, S->s_send);
                        if (nr != ncclSuccess)
                            throw SimError(std::string("ncclSend: ") + S->api->GetErrorString(nr));
                        XK(cudaEventRecord(S->ev_sent[k], S->s_send));
                        if (g_trace) fprintf(stderr, "[ds r%lld] send enqueued c=%lld mb=%d bytes=%lld\n", (long long)s, (long long)c, mb, (long long)bytes);
                    }
                    continue;
                }
                if (NS > 1 && bytes > 0) {
                    // forward hop: the consumer must have read the mb's previous input
                    const int64_t pc = S->prev[c];
                    if (!last && pc >= 0) {
                        {
                            std::unique_lock<std::mutex> lk(next->cs->mu);
                            next->cs->cv.wait(lk, [&] { return next->consumed_c[mb] >= pc || failed.load(); });
                        }
                        if (failed) return;
                        XK(cudaStreamWaitEvent(w.stream, next->consumed_ev[mb], 0));
                    }
                    if (next->device == w.device)
                        XK(cudaMemcpyAsync(next->recv[mb], src, size_t(bytes), cudaMemcpyDeviceToDevice, w.stream));
                    else
                        XK(cudaMemcpyPeerAsync(next->recv[mb], next->device, src, w.device, size_t(bytes), w.stream));
                }
                if (NS == 1) continue;  // nobody waits on the self loop (stream order)
                Mailbox& out = *next->in[mb];
                XK(cudaEventRecord(out.ev, w.stream));
                XK(cudaLaunchHostFunc(w.stream, post_cb, new PostCtx{&out, c, last ? &S->done : nullptr}));
            }
            XK(cudaEventRecord(w.t_end, w.stream));
            XK(cudaStreamSynchronize(w.stream));
        } catch (const std::exception& e) {
            w.error = e.what();
            failed = true;
            for (auto& ww : S->W) {
                for (auto& m : ww.in) m->cv.notify_all();
                ww.cs->cv.notify_all();
            }
            S->land_cv.notify_all();
        }
    };
    // NCCL mode: a receiver thread posts the receives in the previous stage's send order (its
    // compute order, known from the schedule) and publishes each landing to the mailboxes
    auto receiver = [&]() {
        Worker& w = S->W[0];
        try {
            XK(cudaSetDevice(w.device));
            const int64_t from = (w.idx + NS - 1) % NS;
            int64_t posted_n = 0;
            for (const StageOp& op : S->sched.ops[from]) {
                if (failed) return;
                if (op.kind != OpKind::Compute) continue;
                const int64_t c = op.circuit;
                if (c < 0 || c >= S->n_circ) break;
                const size_t bytes = hop_bytes(w.idx, c);
                if (bytes == 0) continue;  // the sender skips empty hops too
                const int32_t mb = circs[c].mb;
                {
                    std::unique_lock<std::mutex> lk(S->land_mu);
                    S->land_cv.wait(lk, [&] { return posted_n - S->landed < Session::kRecvAhead || failed.load(); });
                }
                if (failed) return;
                void* dst = w.recv[mb];
                if (S->ring_mode) {  // slot k: its previous occupant's step must be enqueued
                    const int R = int(S->recv_ring.size());
                    const int k = int(posted_n % R);
                    const int64_t uses = posted_n / R;
                    {
                        std::unique_lock<std::mutex> lk(S->land_mu);
                        S->land_cv.wait(lk, [&] { return S->consumed_n[k] >= uses || failed.load(); });
                    }
                    if (failed) return;
                    if (uses > 0) XK(cudaStreamWaitEvent(S->s_recv, S->ev_consumed[k], 0));
                    S->recv_slot[c] = k;
                    dst = S->recv_ring[k];
                } else if (w.idx > 0 && S->prev[c] >= 0) {  // the mb's previous input must be read first
                    const int64_t pc = S->prev[c];
                    {
                        std::unique_lock<std::mutex> lk(w.cs->mu);
                        w.cs->cv.wait(lk, [&] { return w.consumed_c[mb] >= pc || failed.load(); });
                    }
                    if (failed) return;
                    XK(cudaStreamWaitEvent(S->s_recv, w.consumed_ev[mb], 0));
                }
                const ncclResult_t nr = S->api->Recv(dst, bytes, ncclUint8, 0, S->links.recv, S->s_recv);
                ++posted_n;
                if (nr != ncclSuccess) throw SimError(std::string("ncclRecv: ") + S->api->GetErrorString(nr));
                XK(cudaEventRecord(S->ev_recv[c], S->s_recv));
                XK(cudaLaunchHostFunc(S->s_recv, land_cb, new LandCtx{S}));
                XK(cudaLaunchHostFunc(S->s_recv, post_cb,
                                      new PostCtx{w.in[mb].get(), c, w.idx == 0 ? &S->done : nullptr}));
                if (g_trace) fprintf(stderr, "[ds r%lld] recv posted c=%lld mb=%d bytes=%zu\n", (long long)w.idx, (long long)c, mb, bytes);
            }
            XK(cudaStreamSynchronize(S->s_recv));
        } catch (const std::exception& e) {
            if (w.error.empty()) w.error = std::string("receiver: ") + e.what();
            failed = true;
            for (auto& m : w.in) m->cv.notify_all();
            w.cs->cv.notify_all();
        }
    };
    // NCCL mode watchdog: a local failure, or no landing and no step for DS_NCCL_TIMEOUT_S
    // (default 600 s; the injected hop delays are at most seconds), aborts both link
    // communicators so blocked sends / receives return and the run fails instead of hanging
    std::atomic<bool> done{false};
    std::thread watchdog;
    if (S->nccl) {
        watchdog = std::thread([&]() {
            const char* e = getenv("DS_NCCL_TIMEOUT_S");
            const int64_t limit_us = int64_t(e ? atof(e) : 600.0) * 1000000;
            int64_t last = -1, t_last = now_us();
            while (!done.load()) {
                std::this_thread::sleep_for(std::chrono::milliseconds(200));
                int64_t prog = S->landed;
                for (auto& w : S->W) prog += w.computes;
                if (prog != last) {
                    last = prog;
                    t_last = now_us();
                }
                const bool stalled = now_us() - t_last > limit_us;
                if (failed.load() || stalled) {
                    if (stalled && S->W[0].error.empty())
                        S->W[0].error = "NCCL hop made no progress for DS_NCCL_TIMEOUT_S: aborted";
                    failed = true;
                    S->links.abort(*S->api);
                    S->land_cv.notify_all();
                    for (auto& w : S->W) {
                        for (auto& m : w.in) m->cv.notify_all();
                        w.cs->cv.notify_all();
                    }
                    return;
                }
            }
        });
    }
    std::vector<std::thread> th;
    if (S->nccl) th.emplace_back(receiver);
    for (auto& w : S->W) th.emplace_back(body, std::ref(w));
    for (auto& t : th) t.join();
    done = true;
    if (watchdog.joinable()) watchdog.join();
    if (S->nccl) {
        cudaSetDevice(S->W[0].device);
        cudaStreamSynchronize(S->s_send);
    }
    for (auto& w : S->W) {
        cudaSetDevice(w.device);
        ds_stage_sync(w.st);
    }
    const int64_t t1 = now_us();
    S->t_end = t1;

    GpuRunResult res;
    for (auto& w : S->W)
        if (!w.error.empty() && res.error.empty()) res.error = "stage " + std::to_string(w.idx) + ": " + w.error;
    res.circuits = S->n_circ;
    res.wall_us = t1 - t0;
    for (int64_t c = 0; c < S->n_circ; ++c) {
        res.decode_tokens += circs[c].n_decode;
        res.rows += circs[c].eff_batch;
    }
    int64_t launches1 = 0;
    for (auto& w : S->W) {
        cudaSetDevice(w.device);
        StageRunStats st;
        st.device = w.device;
        st.computes = w.computes;
        st.topups = w.topups;
        st.swap_plan_bytes = w.plan_in;
        st.swap_in_bytes = w.moved_in;
        st.swap_out_bytes = w.moved_out;
        float dev_ms = 0;
        if (res.error.empty() && cudaEventElapsedTime(&dev_ms, w.t_begin, w.t_end) == cudaSuccess)
            st.device_ms = dev_ms;
        res.device_us = std::max<int64_t>(res.device_us, int64_t(double(st.device_ms) * 1000.0));
        for (size_t i = 0; i < w.timing_used; ++i) {
            float ms = 0, wait = 0;
            if (res.error.empty() && cudaEventElapsedTime(&wait, w.timing[i].r, w.timing[i].a) == cudaSuccess)
                res.swap_wait_us += int64_t(double(wait) * 1000.0);
            if (cudaEventElapsedTime(&ms, w.timing[i].a, w.timing[i].b) == cudaSuccess) {
                st.busy_ms += ms;
                st.steps.push_back({w.timing[i].rows, double(ms)});
                float gap = 0;
                if (i > 0 && cudaEventElapsedTime(&gap, w.timing[i - 1].b, w.timing[i].a) == cudaSuccess)
                    st.gaps.push_back(gap);
                else
                    st.gaps.push_back(0.0);
                float end = 0;
                st.ends.push_back(cudaEventElapsedTime(&end, w.t_begin, w.timing[i].b) == cudaSuccess ? end : 0.0);
            }
        }
        std::vector<char> buf(1 << 14);
        int64_t l = 0;
        DK(ds_stage_kernel_stats(w.st, buf.data(), buf.size(), &l));
        st.kernel_stats = buf.data();
        launches1 += l;
        res.stages.push_back(std::move(st));
        res.swaps.push_back(w.swap_pairs);
        const StagePlanD& sp = S->plan.stages[w.idx];
        res.page_bytes.push_back(page_size(S->cfg.model, sp.layer_end - sp.layer_begin, S->cfg.model.num_layers));
    }
    // host -> device bytes of the run: every step's row metadata (kernel_stats "h2d_bytes")
    for (const auto& st : res.stages) {
        const auto p = st.kernel_stats.find("\"h2d_bytes\":");
        if (p != std::string::npos) res.h2d_bytes += std::atoll(st.kernel_stats.c_str() + p + 12);
    }
    res.launches = launches1 - launches0;
    if (collect_tokens && S->tok_pool) {
        res.tokens.resize(S->n_circ);
        for (int64_t c = 0; c < S->n_circ; ++c)
            res.tokens[c].assign(S->tok_pool + S->tok_off[c], S->tok_pool + S->tok_off[c + 1]);
    }
    res.d2h_bytes = collect_tokens ? S->tok_off[S->n_circ] * 4 : 0;
    return res;
}

GpuRunResult run_on_gpus(const Config& cfg, const Plan& plan, const Schedule& sched,
                         const ds_model_desc& md, const GpuOptions& opt) {
    Session* S = session_create(cfg, plan, sched, md, opt);
    GpuRunResult r;
    try {
        r = session_run(S, false, opt.collect_tokens);
    } catch (...) {
        session_destroy(S);
        throw;
    }
    session_destroy(S);
    return r;
}

void session_limit(Session* S, int64_t max_circuits) {
    S->n_circ = max_circuits > 0 ? std::min(max_circuits, S->n_circ_all) : S->n_circ_all;
}
int64_t session_t0(Session* S) { return S->t0; }
int64_t session_end(Session* S) { return S->t_end - S->t0; }
const Config& session_config(Session* S) { return S->cfg; }
const Plan& session_plan(Session* S) { return S->plan; }
int64_t session_vocab(Session* S) { return S->md.vocab; }

void session_capture(Session* S, const std::vector<int64_t>& reqs) {
    S->cap_reqs = reqs;
    std::sort(S->cap_reqs.begin(), S->cap_reqs.end());
}

void session_captured(Session* S, std::vector<int64_t>* meta, const float** logits, int64_t* n) {
    *meta = S->cap_meta;
    *logits = S->cap_pool;
    *n = S->cap_used;
}

std::vector<Record> session_trace(Session* S, int64_t t0_us, bool renumber) {
    if (!S->opt.trace) throw ConfigError("session created without trace recording");
    const int64_t NS = S->plan.S(), NB = S->plan.n_mb;
    const int64_t t0 = t0_us >= 0 ? t0_us : S->t0;
    const auto& circs = S->sched.circuits;
    std::vector<Worker*> wk(NS, nullptr);
    for (auto& w : S->W) wk[w.idx] = &w;
    auto gpu_us = [&](Worker& w, cudaEvent_t e) -> int64_t {
        float ms = 0;
        XK(cudaSetDevice(w.device));
        XK(cudaEventElapsedTime(&ms, w.t_begin, e));
        return w.h_begin + int64_t(double(ms) * 1000.0) - t0;
    };
    // per stage: compute index of each (mb, j-th compute of that mb); swap-op index of each
    // swap with in / out bytes; circuit -> compute index at the last stage
    std::vector<std::vector<std::vector<int64_t>>> comp_of(NS, std::vector<std::vector<int64_t>>(NB));
    std::vector<std::vector<int64_t>> sw_in(NS), sw_out(NS), circ_of(NS);
    std::vector<int64_t> last_comp(circs.size(), -1);
    for (int64_t s = 0; s < NS; ++s) {
        int64_t k = 0, j = 0;
        for (const StageOp& op : S->sched.ops[s]) {
            if (op.kind == OpKind::Compute) {
                comp_of[s][op.mb].push_back(k);
                circ_of[s].push_back(op.circuit);
                if (s == NS - 1 && op.circuit >= 0) last_comp[op.circuit] = k;
                ++k;
            } else if (op.kind == OpKind::SwapIn) {
                if (op.plan_bytes > 0) sw_in[s].push_back(j);
                if (op.evict_bytes > 0) sw_out[s].push_back(j);
                ++j;
            }
        }
    }
    // real times of this process's executed computes
    std::vector<std::vector<int64_t>> t_start(NS), t_end(NS);
    for (int64_t s = 0; s < NS; ++s) {
        Worker* w = wk[s];
        if (!w) continue;
        const size_t n = std::min<size_t>(size_t(w->computes), w->timing_used);
        for (size_t k = 0; k < n; ++k) {
            t_start[s].push_back(gpu_us(*w, w->timing[k].a));
            t_end[s].push_back(gpu_us(*w, w->timing[k].b));
        }
    }
    auto executed = [&](int64_t s, int64_t k) { return wk[s] && k >= 0 && k < int64_t(t_start[s].size()); };
    std::vector<int64_t> cs(NS, 0), ce(NS, 0), si(NS, 0), so(NS, 0);
    std::vector<std::vector<int64_t>> arr_j(NS, std::vector<int64_t>(NB, 0));
    bool have_last = wk[NS - 1] != nullptr, seen_end = false, end_ok = false;
    int64_t end_t = 0;
    std::vector<std::pair<int64_t, Record>> out;  // (virtual seq, event on the real clock)
    for (const Record& e : S->vtrace) {
        Record r = e;
        bool keep = false;
        const int64_t s = e.stage;
        switch (e.kind) {
            case Ev::ComputeStart: {
                const int64_t k = cs[s]++;
                if ((keep = executed(s, k))) r.t = t_start[s][k];
                break;
            }
            case Ev::ComputeEnd: {
                const int64_t k = ce[s]++;
                keep = executed(s, k);
                if (keep) r.t = t_end[s][k];
                if (s == NS - 1) {
                    seen_end = true;
                    end_ok = keep;
                    end_t = r.t;
                }
                break;
            }
            case Ev::TransferArrive: {
                const int64_t j = arr_j[s][e.mb]++;
                if (j >= int64_t(comp_of[s][e.mb].size())) break;
                const int64_t k = comp_of[s][e.mb][j];
                if (!executed(s, k)) break;
                keep = true;
                Worker* w = wk[s];
                if (e.t == 0 && e.a == 0) {
                    r.t = 0;  // initial placement
                } else if (NS == 1) {  // self loop: arrives when its trigger circuit ends
                    const int64_t c = circ_of[s][k];
                    const int64_t trig = c >= 0 ? circs[c].trig : -1;
                    const int64_t tk = trig >= 0 ? last_comp[trig] : -1;
                    if (!executed(0, tk)) { keep = false; break; }
                    r.t = r.a = t_end[0][tk];
                } else {
                    r.t = w->arr_us[k] - t0;
                    r.a = w->send_us[k] - t0;
                }
                break;
            }
            case Ev::SwapInDone:
            case Ev::SwapOutDone: {
                const bool in = e.kind == Ev::SwapInDone;
                const int64_t j = in ? si[s]++ : so[s]++;
                const auto& idx = in ? sw_in[s] : sw_out[s];
                if (j >= int64_t(idx.size()) || !wk[s] || idx[j] >= int64_t(wk[s]->swaps_done)) break;
                const SwapTiming& t = wk[s]->swap_t[idx[j]];
                keep = true;
                r.a = gpu_us(*wk[s], in ? t.e[0] : t.e[2]);
                r.t = gpu_us(*wk[s], in ? t.e[1] : t.e[3]);
                break;
            }
            case Ev::RequestAdmit:
            case Ev::RequestComplete:
                // logged at a last-stage circuit end (or at t=0 before any): that end's time
                if (!have_last) break;
                if (!seen_end) {
                    keep = true;
                    r.t = 0;
                } else if (end_ok) {
                    keep = true;
                    r.t = end_t;
                }
                break;
        }
        if (keep) out.push_back({e.seq, r});
    }
    std::stable_sort(out.begin(), out.end(), [](const auto& x, const auto& y) {
        return x.second.t != y.second.t ? x.second.t < y.second.t : x.first < y.first;
    });
    std::vector<Record> tr;
    tr.reserve(out.size());
    for (size_t i = 0; i < out.size(); ++i) {
        tr.push_back(out[i].second);
        tr.back().seq = renumber ? int64_t(i) : out[i].first;
    }
    return tr;
}

std::string GpuRunResult::to_json() const {
    std::ostringstream os;
    os.precision(10);
    os << "{\"circuits\":" << circuits << ",\"decode_tokens\":" << decode_tokens << ",\"rows\":" << rows
       << ",\"wall_us\":" << wall_us << ",\"device_us\":" << device_us << ",\"launches\":" << launches
       << ",\"d2h_bytes\":" << d2h_bytes << ",\"h2d_bytes\":" << h2d_bytes
       << ",\"swap_wait_us\":" << swap_wait_us << ",\"page_bytes\":[";
    for (size_t i = 0; i < page_bytes.size(); ++i) os << (i ? "," : "") << page_bytes[i];
    os << "],\"swap_pairs\":[";  // per stage: [plan, slot refill, migration, eviction] per swap-in
    for (size_t i = 0; i < swaps.size(); ++i) {
        os << (i ? ",[" : "[");
        for (size_t k = 0; k < swaps[i].size(); ++k)
            os << (k ? ",[" : "[") << swaps[i][k].plan << "," << swaps[i][k].slot_in << ","
               << swaps[i][k].migrated << "," << swaps[i][k].moved_out << "]";
        os << "]";
    }
    os << "],\"tokens_per_s\":"
       << (wall_us > 0 ? double(decode_tokens) * 1e6 / double(wall_us) : 0.0) << ",\"error\":\"";
    for (char ch : error) os << (ch == '"' || ch == '\\' ? ' ' : ch);
    os << "\",\"stages\":[";
    for (size_t i = 0; i < stages.size(); ++i) {
        const auto& s = stages[i];
        os << (i ? "," : "") << "{\"device\":" << s.device << ",\"computes\":" << s.computes
           << ",\"busy_ms\":" << s.busy_ms << ",\"device_ms\":" << s.device_ms << ",\"topups\":" << s.topups
           << ",\"swap_plan_bytes\":" << s.swap_plan_bytes << ",\"swap_in_bytes\":" << s.swap_in_bytes
           << ",\"swap_out_bytes\":" << s.swap_out_bytes << ",\"kernels\":"
           << (s.kernel_stats.empty() ? "{}" : s.kernel_stats) << ",\"steps\":[";
        for (size_t k = 0; k < s.steps.size(); ++k)
            os << (k ? "," : "") << "[" << s.steps[k].first << "," << s.steps[k].second << ","
               << (k < s.gaps.size() ? s.gaps[k] : 0.0) << "," << (k < s.ends.size() ? s.ends[k] : 0.0)
               << "]";
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
