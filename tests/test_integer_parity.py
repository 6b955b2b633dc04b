"""Integer hot path: the product's planner / perf model / scheduler against
(1) the reference's own unit-test goldens and (2) the compiled reference (oracle/_ref), bit-exact.
CPU only."""
import hashlib
import json
import os
import sys

import pytest

from paper_2501_14784_b200 import pipeline as pl
from paper_2501_14784_b200._native import PlanError, SimError

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
GOLD = json.load(open(os.path.join(ROOT, "tests", "golden", "reference_unit_goldens.json")))
CONFIGS = os.path.join(ROOT, "configs")
REF_CONFIGS = os.path.join(ROOT, "tests", "golden", "ref_configs")
GIB = 1 << 30


@pytest.fixture(scope="module")
def ref():
    import oracle
    return oracle.Ref()


def sha(path):
    return hashlib.sha256(open(path, "rb").read()).hexdigest()


# ------------------------------------------------------------------- unit-test goldens ----
def test_stage_time_goldens(ref):
    tab = GOLD["stage_time_points"]["table1"]
    for b, us in tab:
        assert pl.stage_time_us(tab, b, 1, 0) == us == ref.stage_time(tab, b, 1, 0)
    for b, us in GOLD["stage_time_interp"]["cases"]:
        assert pl.stage_time_us(tab, b, 1, 0) == us == ref.stage_time(tab, b, 1, 0)
    small = GOLD["stage_time_clamp"]["table"]
    for b, us in GOLD["stage_time_clamp"]["cases"]:
        assert pl.stage_time_us(small, b, 1, 0) == us
    for b, layers, refl, us in GOLD["scaled_stage_time"]["cases"]:
        assert pl.stage_time_us(tab, b, layers, refl) == us == ref.stage_time(tab, b, layers, refl)


def test_stage_time_exhaustive_vs_reference(ref):
    tabs = [GOLD["stage_time_points"]["table1"], [[1, 2000], [64, 5000], [512, 20000]],
            [[3, 17], [5, 17], [9, 1000], [100, 100001]]]
    for tab in tabs:
        for b in range(1, 700):
            for layers, refl in [(1, 0), (10, 10), (7, 3), (40, 80), (3, 7)]:
                assert pl.stage_time_us(tab, b, layers, refl) == ref.stage_time(tab, b, layers, refl)


def test_page_and_pool_goldens(ref):
    g = GOLD["page_bytes_70b"]
    for layers, total, want in g["cases"]:
        assert pl.page_bytes(g["kv_bytes_per_token"], layers, total) == want
        assert ref.page_bytes(g["kv_bytes_per_token"], layers, total) == want
    for w, t, page, want in GOLD["global_pool_size"]["cases"]:
        assert pl.global_pool_size(w, t, page) == want == ref.global_pool_size(w, t, page)
    for kv in [2048, 131072, 327680, 8192 * 3, 1]:
        for total in [1, 4, 32, 80]:
            for layers in range(1, total + 1, max(1, total // 7)):
                assert pl.page_bytes(kv, layers, total) == ref.page_bytes(kv, layers, total)


def test_memory_budget_grid(ref):
    for m, w, nb, g, mb, mbo in GOLD["memory_budget_grid"]["rows"]:
        out = pl.memory_budget(m, w, nb, g, True)
        assert out[0] == m - w and out[2] == mb and out[3] == mbo
        assert out == ref.memory_budget(m, w, nb, g, True)
        plain = pl.memory_budget(m, w, nb, g, False)
        assert plain[1] == 0 and plain[3] == mb
        assert plain == ref.memory_budget(m, w, nb, g, False)


def test_memory_budget_errors():
    with pytest.raises(PlanError):
        pl.memory_budget(8 * GIB, 9 * GIB, 4, 0, False)
    with pytest.raises(PlanError):
        pl.memory_budget(8 * GIB, 4 * GIB, 4, 3 * GIB, True)


def test_request_generator_matches_reference(ref):
    for seed in [0, 7, 42, 2 ** 63 + 5]:
        for rng in [(0, 512, 0, 512), (7, 7, 3, 3), (3840, 3840, 256, 256), (0, 1, 0, 1)]:
            for k in list(range(50)) + [10 ** 6, 2 ** 40]:
                assert pl.request_lengths(seed, *rng, k) == ref.request(seed, *rng, k)
    vals = [pl.request_lengths(42, 0, 512, 0, 512, k) for k in range(100000)]
    mp = sum(v[0] for v in vals) / len(vals)
    mo = sum(v[1] for v in vals) / len(vals)
    assert 251 < mp < 261 and 251 < mo < 261  # test_workload.cpp:25-42


def ring_config(n, mem, pcie, latency, bw, policy=None, workload=None):
    nodes = [{"node_id": f"n{i}", "gpu_mem_bytes": mem, "pcie_bandwidth_bytes_per_s": pcie,
              "compute_calibration": "table1"} for i in range(n)]
    links = [{"src": f"n{i}", "dst": f"n{(i + 1) % n}", "latency_us": latency,
              "bandwidth_bytes_per_s": bw} for i in range(n)] if n > 1 else []
    wl = workload or {"prompt_len_min": 0, "prompt_len_max": 512, "output_len_min": 0,
                      "output_len_max": 512, "concurrency_target": 2048, "bench_duration_s": 1200,
                      "warmup_s": 240, "rng_seed": 42}
    cfg = {"model": "llama3-70b", "nodes": nodes, "links": links, "workload": wl}
    if policy:
        cfg["scheduler"] = policy
    return json.dumps(cfg)


def test_planner_golden(ref):
    g = GOLD["planner_golden"]
    txt = ring_config(8, 24 * GIB, g["pcie"], g["latency_us"], g["bw"],
                      {"offload": True, "calibration_ref_layers": 10})
    mine = pl.plan_config(txt)
    assert mine == ref.plan_config(txt)
    p = json.loads(mine)
    assert p["converged"] and p["iterations"] == g["iterations"]
    assert p["stages"][0]["batch_size_per_microbatch"] == g["batch"]
    assert p["n_microbatches"] == g["n_microbatches"] and p["stage_time_us"] == g["stage_time_us"]
    assert all(s["budget"]["m_global_pool"] == g["m_global_pool"] for s in p["stages"])
    assert p["stages"][0]["budget"]["m_kv"] == g["m_kv_stage0"]
    assert p["stages"][1]["budget"]["m_kv"] == g["m_kv_stage1"]
    assert [[s["layer_begin"], s["layer_end"]] for s in p["stages"]] == [[10 * i, 10 * i + 10] for i in range(8)]


def test_planner_partitions_and_errors(ref):
    txt = ring_config(2, 96 * GIB, 16 * 10 ** 9, 1000, 10 ** 9, {"offload": False})
    p = json.loads(pl.plan_config(txt))
    assert [[s["layer_begin"], s["layer_end"]] for s in p["stages"]] == GOLD["planner_partition"]["sym2_96gib"]
    cfg = json.loads(ring_config(2, 120 * GIB, 16 * 10 ** 9, 1000, 10 ** 9, {"offload": False}))
    cfg["nodes"][1]["gpu_mem_bytes"] = 40 * GIB
    p = json.loads(pl.plan_config(json.dumps(cfg)))
    assert [[s["layer_begin"], s["layer_end"]] for s in p["stages"]] == GOLD["planner_partition"]["big_small"]
    assert pl.plan_config(json.dumps(cfg)) == ref.plan_config(json.dumps(cfg))
    with pytest.raises(PlanError, match="insufficient-total-memory"):
        pl.plan_config(ring_config(2, 24 * GIB, 16 * 10 ** 9, 1000, 10 ** 9))
    broken = json.loads(ring_config(8, 24 * GIB, 32 * 10 ** 9, 64000, 10 ** 9, {"nb_override": 5}))
    broken["links"].pop()
    with pytest.raises(PlanError, match="missing-link"):
        pl.plan_config(json.dumps(broken))
    big = json.loads(ring_config(8, 24 * GIB, 32 * 10 ** 9, 64000, 10 ** 9))
    big["workload"]["prompt_len_max"] = big["workload"]["output_len_max"] = 4000
    with pytest.raises(PlanError, match="max_seq_len"):
        pl.plan_config(json.dumps(big))


@pytest.mark.parametrize("S,lat,t_s,want", [(4, 35000, 70000, 6), (4, 61728, 123456, 6), (8, 64000, 70000, 16)])
def test_min_bubble_free(S, lat, t_s, want):
    # N_B = S + ceil(S*L/T_S) (planner.cpp:80-91), through the planner with a flat calibration
    cfg = json.loads(ring_config(S, 96 * GIB, 16 * 10 ** 9, lat, 10 ** 12, {"offload": False}))
    open("/tmp/flat_cal.csv", "w").write(f"1,{t_s / 1000:.3f}\n100000,{t_s / 1000:.3f}\n")
    for n in cfg["nodes"]:
        n["compute_calibration"] = "/tmp/flat_cal.csv"
    assert json.loads(pl.plan_config(json.dumps(cfg)))["n_microbatches"] == want


# ---------------------------------------------------------- schedule / swap-plan parity ----
def _short(cfg_path, duration=None, warmup=None):
    cfg = json.load(open(cfg_path))
    if duration:
        cfg["workload"]["bench_duration_s"] = duration
        cfg["workload"]["warmup_s"] = warmup
    return json.dumps(cfg)


REF8 = "/root/reference/proj/configs/reference_8stage.json"
RING4 = "/root/reference/proj/configs/fig_ring4.json"


def _ref_config(name):
    """The reference's shipped configs; committed copies keep the test runnable off-container."""
    p = os.path.join("/root/reference/proj/configs", name)
    return p if os.path.exists(p) else os.path.join(REF_CONFIGS, name)


@pytest.mark.parametrize("policy", ["baseline", "offload", "opt"])
@pytest.mark.parametrize("latency", [0, 16000, 64000, 256000])
def test_reference_8stage_trace_identical(ref, tmp_path, policy, latency):
    txt = _short(_ref_config("reference_8stage.json"), 300, 60)
    assert pl.plan_config(txt, "", policy, latency) == ref.plan_config(txt, "", policy, latency)
    a, b = str(tmp_path / "a.tr"), str(tmp_path / "b.tr")
    ra = pl.sim_config(txt, "", policy, latency, trace_path=a)
    rb = ref.sim_config(txt, "", policy, latency, trace_path=b)
    assert ra == rb
    assert sha(a) == sha(b)
    plan = pl.plan_config(txt, "", policy, latency)
    assert ref.replay_check(a, plan) == []
    assert ref.windowed_stats(a, ra["window_start_us"], ra["window_end_us"])[1] == ra["output_tokens"]


@pytest.mark.parametrize("policy,latency", [("baseline", 0), ("baseline", 35150), ("opt", 35150), ("offload", 35150)])
def test_fig_ring4_trace_identical(ref, tmp_path, policy, latency):
    txt = _short(_ref_config("fig_ring4.json"), 200, 40)
    a, b = str(tmp_path / "a.tr"), str(tmp_path / "b.tr")
    assert pl.sim_config(txt, "", policy, latency, trace_path=a) == ref.sim_config(txt, "", policy, latency, trace_path=b)
    assert sha(a) == sha(b)


@pytest.mark.parametrize("name", ["tiny_2stage.json", "tiny_2stage_swap.json", "llama8b_1stage.json",
                                  "llama8b_4stage.json", "llama8b_4stage_swap.json",
                                  "llama70b_8stage.json", "llama70b_8stage_swap.json"])
def test_baseline_configs_trace_identical(ref, tmp_path, name):
    path = os.path.join(CONFIGS, name)
    cfg = json.load(open(path))
    if cfg["workload"]["bench_duration_s"] > 120:
        cfg["workload"]["bench_duration_s"] = 120
    txt = json.dumps(cfg)
    assert pl.plan_config(txt, CONFIGS) == ref.plan_config(txt, CONFIGS)
    a, b = str(tmp_path / "a.tr"), str(tmp_path / "b.tr")
    ra = pl.sim_config(txt, CONFIGS, trace_path=a)
    assert ra == ref.sim_config(txt, CONFIGS, trace_path=b)
    assert sha(a) == sha(b)
    assert ref.replay_check(a, pl.plan_config(txt, CONFIGS)) == []


def decode_ring(s, nb, b, hop, concurrency=-1):
    """tests/fixtures.hpp:20-72 as (config, plan) documents."""
    table1 = GOLD["stage_time_points"]["table1"]
    t_s = pl.stage_time_us(table1, b, 1, 0)
    mem = 1 << 40
    nodes = [{"node_id": f"n{i}", "gpu_mem_bytes": mem, "pcie_bandwidth_bytes_per_s": 32_000_000_000,
              "compute_calibration": "table1"} for i in range(s)]
    links = [{"src": f"n{i}", "dst": f"n{(i + 1) % s}", "latency_us": hop,
              "bandwidth_bytes_per_s": 1_000_000_000_000} for i in range(s)] if s > 1 else []
    period = max(nb * t_s, s * t_s + s * hop)
    warm = 10 * period // 1_000_000 + 1
    cfg = {"model": {"name": "synthetic", "num_layers": s, "weight_bytes_total": 2 + s,
                     "embedding_bytes": 1, "output_layer_bytes": 1, "kv_bytes_per_token": 8192 * s,
                     "max_seq_len": 1_000_000_000},
           "nodes": nodes, "links": links,
           "workload": {"prompt_len_min": 0, "prompt_len_max": 0, "output_len_min": 900_000_000,
                        "output_len_max": 900_000_000,
                        "concurrency_target": nb * b if concurrency < 0 else concurrency,
                        "bench_duration_s": warm + 100 * period // 1_000_000 + 1, "warmup_s": warm,
                        "rng_seed": 7}}
    bud = pl.memory_budget(mem, 1, nb, 0, False)
    plan = {"n_microbatches": nb, "stage_time_us": t_s, "offload_enabled": False, "converged": True,
            "iterations": 0, "seq_budget_tokens": 1_000_000_000,
            "policy": {"offload": False, "nb_override": 0, "prefill_chunk": 256,
                       "hidden_bytes_per_token": 0, "kv_reserve_permille": 300,
                       "calibration_ref_layers": 0, "ring_order": "config", "pool_scale_milli": 1000,
                       "pool_time_basis": "compute"},
            "stages": [{"node_id": f"n{i}", "layer_begin": i, "layer_end": i + 1, "stage_weight_bytes": 1,
                        "pcie_bandwidth_bytes_per_s": 32_000_000_000, "batch_size_per_microbatch": b,
                        "stage_time_us": t_s,
                        "budget": {"m_total": mem, "m_weights": 1, "m_kv": bud[0], "m_global_pool": 0,
                                   "n_microbatches": nb, "m_per_microbatch_no_offload": bud[2],
                                   "m_per_microbatch_offload": bud[3], "offload": False}}
                       for i in range(s)],
            "ring_links": json.loads(json.dumps(links))}
    return cfg, plan


@pytest.mark.parametrize("s,nb,b,hop", [(1, 1, 32, 0), (4, 4, 16, 35150), (4, 6, 16, 35150), (2, 2, 8, 0),
                                        (2, 5, 24, 100000), (3, 7, 12, 50000), (5, 9, 40, 20000),
                                        (8, 16, 20, 64000), (8, 8, 64, 5000), (6, 24, 16, 250000)])
def test_decode_ring_fixtures(ref, tmp_path, s, nb, b, hop):
    cfg, plan = decode_ring(s, nb, b, hop)
    txt, pj = json.dumps(cfg), json.dumps(plan)
    a, bpath = str(tmp_path / "a.tr"), str(tmp_path / "b.tr")
    ra = pl.sim_plan(txt, pj, trace_path=a)
    assert ra == ref.sim_plan(txt, pj, trace_path=bpath)
    assert sha(a) == sha(bpath)
    # analytic oracle within 2% (test_sim.cpp:66-86)
    assert abs(ra["output_throughput"] - pl.steady_state_throughput(pj)) <= 0.02 * pl.steady_state_throughput(pj)
    assert pl.steady_state_throughput(pj) == pytest.approx(ref.steady_state(pj), rel=1e-15)


def test_decode_ring_closed_forms():
    cfg, plan = decode_ring(1, 1, 32, 0)
    r = pl.sim_plan(json.dumps(cfg), json.dumps(plan))
    assert r["output_throughput"] == pytest.approx(32e6 / 76500, rel=0.01)  # test_sim.cpp:23-31
    cfg, plan = decode_ring(4, 4, 16, 35150)
    r = pl.sim_plan(json.dumps(cfg), json.dumps(plan))
    for st in r["stages"]:  # test_sim.cpp:33-44
        assert st["bubble_fraction"] == pytest.approx(1 / 3, rel=0.01)
        assert st["transfer_wait_fraction"] == 0


def test_conservation_and_zero_work(ref, tmp_path):
    cfg, plan = decode_ring(3, 4, 8, 10000)
    cfg["workload"].update(output_len_min=40, output_len_max=40, prompt_len_min=10, prompt_len_max=10,
                           concurrency_target=64, bench_duration_s=120, warmup_s=10)
    a, b = str(tmp_path / "a.tr"), str(tmp_path / "b.tr")
    r = pl.sim_plan(json.dumps(cfg), json.dumps(plan), trace_path=a)
    assert r == ref.sim_plan(json.dumps(cfg), json.dumps(plan), trace_path=b) and sha(a) == sha(b)
    assert r["live_requests"] <= 64 and r["completed_requests"] > 0
    cfg, plan = decode_ring(2, 2, 4, 1000)
    cfg["workload"].update(prompt_len_min=0, prompt_len_max=1, output_len_min=0, output_len_max=1,
                           concurrency_target=32, bench_duration_s=30, warmup_s=2)
    r = pl.sim_plan(json.dumps(cfg), json.dumps(plan), trace_path=a)
    assert r == ref.sim_plan(json.dumps(cfg), json.dumps(plan), trace_path=b) and sha(a) == sha(b)
    assert r["completed_requests"] > 0


def test_plan_topology_mismatch():
    cfg, plan = decode_ring(3, 3, 8, 1000)
    cfg["links"][0]["latency_us"] += 5
    with pytest.raises(SimError, match="mismatch"):
        pl.sim_plan(json.dumps(cfg), json.dumps(plan))


# ------------------------------------------------------- report recomputed from a trace ----
@pytest.mark.parametrize("name,policy,latency", [
    ("configs/tiny_2stage_swap.json", None, -1), ("configs/llama8b_4stage_swap.json", None, -1),
    ("tests/golden/ref_configs/reference_8stage.json", "opt", 64000),
    ("tests/golden/ref_configs/reference_8stage.json", "offload", 16000),
    ("tests/golden/ref_configs/reference_8stage.json", "baseline", 256000),
    ("tests/golden/ref_configs/fig_ring4.json", None, -1)])
def test_trace_report_equals_reference_run(ref, tmp_path, name, policy, latency):
    """ds_trace_report (the report of hardware runs, computed from their trace) reproduces the
    reference run()'s SimReport (build_report, sim.cpp:501-532 -- including per-stage busy, swap
    stall and bubble) from the reference's own trace of the same run."""
    path = os.path.join(ROOT, name)
    txt, cdir = open(path).read(), os.path.dirname(path)
    tr = str(tmp_path / "ref.trace")
    want = ref.sim_config(txt, cdir, policy=policy, latency_us=latency, trace_path=tr)
    cfg = json.loads(txt)
    wl = cfg["workload"]
    n_stages = len(json.loads(ref.plan_config(txt, cdir, policy=policy, latency_us=latency))["stages"])
    got = pl.trace_report(tr, n_stages, wl["warmup_s"] * 10**6, wl["bench_duration_s"] * 10**6,
                          wl["rng_seed"])
    for k in ("input_tokens", "output_tokens", "completed_requests", "admitted_requests",
              "live_requests", "swap_stall_us", "window_start_us", "window_end_us"):
        assert got[k] == want[k], k
    for a, b in zip(got["stages"], want["stages"]):
        assert (a["busy_us"], a["stall_us"], a["bubble_us"]) == (b["busy_us"], b["stall_us"],
                                                                 b["bubble_us"])
    assert got["output_throughput"] == pytest.approx(want["output_throughput"], rel=1e-12)


def test_trace_merge_orders_rank_traces(tmp_path):
    """Per-rank traces (virtual seq kept) merge into one (time, seq)-ordered trace."""
    cfg = os.path.join(CONFIGS, "tiny_2stage.json")
    txt = open(cfg).read()
    full = str(tmp_path / "full.trace")
    pl.sim_config(txt, CONFIGS, trace_path=full)
    lines = open(full).read().splitlines()
    parts = [str(tmp_path / f"r{i}.trace") for i in range(2)]
    # split by stage parity (stage -1 events with rank 1), as two ranks would write them
    with open(parts[0], "w") as a, open(parts[1], "w") as b:
        for ln in lines:
            st = int(ln.split("stage=")[1].split()[0])
            (a if st == 0 else b).write(ln + "\n")
    merged = str(tmp_path / "m.trace")
    pl.trace_merge(parts, merged)
    assert open(merged).read() == open(full).read()


@pytest.mark.parametrize("policy,latency", [("opt", 64000), ("baseline", 16000), ("offload", 256000)])
def test_report_kv_identical(ref, policy, latency):
    """report.kv of our run (ds_report_kv) is byte-identical to the reference's report_to_kv
    (src/sweep.cpp:146-195) of the same cell."""
    path = os.path.join(REF_CONFIGS, "reference_8stage.json")
    txt = open(path).read()
    rep = pl.sim_config(txt, REF_CONFIGS, policy=policy, latency_us=latency)
    plan = pl.plan_config(txt, REF_CONFIGS, policy=policy, latency_us=latency)
    assert pl.report_kv(rep, plan, latency, policy) == ref.report_kv(txt, REF_CONFIGS, policy, latency)


def test_sweep_csv_identical(ref):
    """sweep.csv of our latency x policy matrix (ds_sweep_csv) is byte-identical to the reference's
    run_sweep(...).to_csv() (src/sweep.cpp:68-82,101-144)."""
    path = os.path.join(REF_CONFIGS, "reference_8stage.json")
    txt = open(path).read()
    lats = json.loads(txt)["sweep"]["latencies_us"]
    pols = ["baseline", "offload", "opt"]
    tput = [[pl.sim_config(txt, REF_CONFIGS, policy=p, latency_us=l)["output_throughput"] for l in lats]
            for p in pols]
    assert pl.sweep_csv(lats, pols, tput) == ref.sweep_csv(txt, REF_CONFIGS)


def test_reference_binding_links_and_maps_errors(tmp_path):
    """The reference-side binding (integration/run_on_b200.cpp) compiles against the reference
    headers and links both libraries; without a GPU the product's no-device error reaches the
    caller as pipesim::SimError text (no CPU fallback)."""
    import oracle
    from paper_2501_14784_b200 import n_devices
    from paper_2501_14784_b200._native import GpuOpts
    if n_devices() > 0:
        pytest.skip("GPU present: tests/test_gpu_trace.py runs the binding end to end")
    txt = open(os.path.join(CONFIGS, "tiny_2stage.json")).read()
    opts = GpuOpts(device0=0, n_devices=1, real_delay=1, collect_tokens=0, max_circuits=4,
                   weight_seed=pl.WEIGHT_SEED, trace=1)
    with pytest.raises(oracle.RefError, match="CUDA device"):
        oracle.binding_run_and_check(txt, CONFIGS, pl.plan_config(txt, CONFIGS),
                                     pl.model_desc("tiny-llama"), opts, str(tmp_path / "t.trace"))


PRICINGS = [
    {"preset": "whattomine-8x4090"}, {"preset": "gcp-8xL4"}, {"preset": "runpod-8x4090"},
    {"preset": "ionet-8x4090"},
    {"compute_cost_per_hour": 2.5, "price_per_token": 0.0000009},
    {"compute_cost_per_hour": 13.878, "price_per_token": 0.0000002,
     "price_in_per_token": 0.0000001, "price_out_per_token": 0.0000004},
    {"compute_cost_per_hour": 40.0, "price_per_token": 0.00000001},  # unprofitable
]


@pytest.mark.parametrize("pricing", PRICINGS)
@pytest.mark.parametrize("policy,latency", [("opt", 64000), ("baseline", 16000)])
def test_priced_report_kv_identical(ref, pricing, policy, latency):
    """report.kv with the profit block (ds_report_kv_priced: economics.cpp restated) is
    byte-identical to the reference's report_to_kv(report, plan, latency, policy, &analyze(...))
    for presets, unified and split prices, profitable or not."""
    cfg = json.load(open(os.path.join(REF_CONFIGS, "reference_8stage.json")))
    cfg["pricing"] = pricing
    txt = json.dumps(cfg)
    rep = pl.sim_config(txt, REF_CONFIGS, policy=policy, latency_us=latency)
    plan = pl.plan_config(txt, REF_CONFIGS, policy=policy, latency_us=latency)
    ours = pl.report_kv(rep, plan, latency, policy, pricing)
    assert ours == ref.report_kv_priced(txt, REF_CONFIGS, policy, latency)
    assert ours.startswith(pl.report_kv(rep, plan, latency, policy)) and "profitable=" in ours


@pytest.mark.parametrize("pricing,msg", [
    ({"preset": "nope"}, "unknown pricing preset"),
    ({"preset": "gcp-8xL4", "price_per_token": 1}, "unknown field"),
    ({"compute_cost_per_hour": 1.0}, "no price fields"),
    ({"compute_cost_per_hour": 1.0000001, "price_per_token": 0.000001}, "finer than"),
    ({"compute_cost_per_hour": 1.0, "price_in_per_token": 0.000001}, "positive price per token"),
])
def test_priced_report_kv_errors(ref, pricing, msg):
    """Pricing errors as the reference raises them: config parsing (config.cpp:169-199) and
    analyze's zero unified price (economics.cpp:16-20: split prices without price_per_token)."""
    cfg = json.load(open(os.path.join(REF_CONFIGS, "reference_8stage.json")))
    cfg["pricing"] = pricing
    txt = json.dumps(cfg)
    rep = pl.sim_config(json.dumps(dict(cfg, pricing={"preset": "gcp-8xL4"})), REF_CONFIGS)
    plan = pl.plan_config(json.dumps(dict(cfg, pricing={"preset": "gcp-8xL4"})), REF_CONFIGS)
    with pytest.raises(Exception, match=msg):
        pl.report_kv(rep, plan, 0, "config", pricing)
    with pytest.raises(Exception, match=msg):
        ref.report_kv_priced(txt, REF_CONFIGS)


@pytest.mark.parametrize("run", ["r02_70b_8stage_4gpu", "r02_8b_4stage_swap_pin",
                                 "r02_70b_4stage_swap_pin"])
def test_hardware_runs_repriced(tmp_path, run):
    """Economics on GPU runs: the committed real-clock hardware trace of a B200 run rebuilds its
    committed report.kv byte for byte (ds_trace_report), and the priced report appends the
    reference's profit block (tools/price_runs.py; profiles/<run>/report_priced.kv)."""
    sys.path.insert(0, os.path.join(ROOT, "tools"))
    import price_runs
    d = os.path.join(ROOT, "profiles", run)
    out = price_runs.price_run(d, {"preset": "whattomine-8x4090"}, out_dir=str(tmp_path))
    assert out["profitable"] == "1" and int(out["revenue_micro_usd"]) > int(out["cost_micro_usd"])
    assert open(tmp_path / "report_priced.kv").read() == open(os.path.join(d, "report_priced.kv")).read()


def _write_trace(lines, path):
    """Trace lines with seq renumbered to the line index (write_trace's invariant)."""
    with open(path, "w") as f:
        for i, ln in enumerate(lines):
            fs = ln.split()
            fs[1] = f"seq={i}"
            f.write(" ".join(fs) + "\n")


def test_committed_hardware_trace_passes_and_tampering_is_caught(ref, tmp_path):
    """The reference's replay_check (sim.cpp:606-697) on a committed B200 hardware trace (70B,
    8 stages on 4 GPUs): 0 violations; the same trace with one compute duplicated, or with a hop
    arriving before the compute that sends it, is rejected -- the gate is live, not vacuous."""
    import gzip
    d = os.path.join(ROOT, "profiles", "r02_70b_8stage_4gpu")
    s = json.load(open(os.path.join(d, "summary.json")))
    plan = pl.plan_config(open(os.path.join(ROOT, s["config"])).read(), os.path.join(ROOT, "configs"))
    lines = gzip.open(os.path.join(d, "hw.trace.gz"), "rt").read().splitlines()
    clean = str(tmp_path / "clean.trace")
    _write_trace(lines, clean)
    assert ref.replay_check(clean, plan) == []
    # double compute: a second ComputeStart of stage 1's first compute
    i = next(k for k, ln in enumerate(lines) if "kind=ComputeStart stage=1 " in ln)
    dup = str(tmp_path / "dup.trace")
    _write_trace(lines[:i + 1] + [lines[i]] + lines[i + 1:], dup)
    assert ref.replay_check(dup, plan) != []
    # causality: stage 1's first arrival moved to t=1 (t=0 marks initial placements), before its
    # send time + hop latency
    j = next(k for k, ln in enumerate(lines) if "kind=TransferArrive stage=1 " in ln)
    early = lines[:j] + [" ".join(["t=1"] + lines[j].split()[1:])] + lines[j + 1:]
    bad = str(tmp_path / "early.trace")
    _write_trace(early, bad)
    assert ref.replay_check(bad, plan) != []


def _committed_runs():
    base = os.path.join(ROOT, "profiles")
    return sorted(d for d in os.listdir(base) if os.path.exists(os.path.join(base, d, "hw.trace.gz")))


@pytest.mark.parametrize("run", _committed_runs())
def test_every_committed_hardware_trace_replays_clean(ref, tmp_path, run):
    """Every committed real-clock B200 trace under profiles/ passes the reference's replay_check
    against its plan, except the one rule DESIGN.md section 9 explains: swap-bandwidth-exceeded
    (SwapIn/OutDone carry the plan's bytes while the copies move only the occupied tokens of
    partial pages, so they finish sooner than plan_bytes / modelled link rate)."""
    import gzip
    sys.path.insert(0, ROOT)
    import bench_multi
    d = os.path.join(ROOT, "profiles", run)
    cdir = os.path.join(ROOT, "configs")
    if os.path.exists(os.path.join(d, "summary.json")):
        s = json.load(open(os.path.join(d, "summary.json")))
        txt, pol = open(os.path.join(ROOT, s["config"])).read(), s.get("policy")
        plan = pl.plan_config(txt, cdir, policy=pol, latency_us=s["latency_us"] if pol else -1)
    else:  # bench.py --gpus N run: BASELINE configs[2] with N nodes
        kv = dict(ln.split("=", 1) for ln in open(os.path.join(d, "report.kv")).read().splitlines())
        plan = pl.plan_config(json.dumps(bench_multi.pipeline_config(int(kv["n_stages"]))), cdir)
    trace = tmp_path / "hw.trace"
    trace.write_text(gzip.open(os.path.join(d, "hw.trace.gz"), "rt").read())
    kinds = {v.split()[0] for v in ref.replay_check(str(trace), plan)}
    assert kinds <= {"swap-bandwidth-exceeded"}
    # and the reference's windowed_stats (workload.cpp:82-116) over the report's window counts
    # exactly the committed report's tokens: the headline numbers are the reference metric
    kv = dict(ln.split("=", 1) for ln in open(os.path.join(d, "report.kv")).read().splitlines())
    n_in, n_out, _ = ref.windowed_stats(str(trace), int(kv["window_start_us"]), int(kv["window_end_us"]))
    assert (n_in, n_out) == (int(kv["input_tokens"]), int(kv["output_tokens"]))


def test_committed_gpu_sweep_is_against_the_reference_sweep(ref):
    """profiles/r02_sweep_70b (config 5 on 4 B200s, tools/gpu_sweep.py --duration 60 --warmup 20):
    its sweep_reference.csv is the reference's own run_sweep(...).to_csv() of the same document,
    and sweep_gpu.csv (ds_sweep_csv) holds the per-cell hardware throughputs of cells.jsonl."""
    d = os.path.join(ROOT, "profiles", "r02_sweep_70b")
    cfg = json.load(open(os.path.join(ROOT, "configs", "llama70b_sweep_4gpu.json")))
    cfg["workload"].update(bench_duration_s=60, warmup_s=20)
    assert open(os.path.join(d, "sweep_reference.csv")).read() == \
        ref.sweep_csv(json.dumps(cfg), os.path.join(ROOT, "configs"))
    cells = [json.loads(ln) for ln in open(os.path.join(d, "cells.jsonl"))]
    rows = {ln.split(",")[0]: ln.strip().split(",")[1:]
            for ln in open(os.path.join(d, "sweep_gpu.csv")).read().splitlines()[1:]}
    lats = open(os.path.join(d, "sweep_gpu.csv")).readline().strip().split(",")[1:]
    for c in cells:
        assert c["replay_check"]["violations"] == 0
        got = float(rows[c["policy"]][lats.index(str(c["latency_us"]))])
        assert abs(got - c["gpu_tps"]) <= 0.06
