"""CPU checks of bench.py's measurement legs (no GPU): the schedule fixture the reference arm
times is the reference's own schedule, and the reference arm never loads the product library."""
import gzip
import json
import os
import subprocess
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
CONFIGS = os.path.join(ROOT, "configs")


def test_schedule_fixture_is_the_reference_schedule(tmp_path):
    """configs/llama8b_1stage.schedule.json.gz (tools/make_schedule_fixture.py): every circuit's
    (eff_batch, n_decode) equals the ComputeStart events of the reference's own run() trace of
    configs/llama8b_1stage.json (oracle/_ref), and its rows add up to them."""
    import oracle
    fx = json.load(gzip.open(os.path.join(CONFIGS, "llama8b_1stage.schedule.json.gz"), "rt"))
    txt = open(os.path.join(CONFIGS, "llama8b_1stage.json")).read()
    tr = str(tmp_path / "ref.trace")
    oracle.Ref().sim_config(txt, CONFIGS, trace_path=tr)
    starts = []
    for line in open(tr):
        if "kind=ComputeStart" in line:
            f = dict(x.split("=", 1) for x in line.split())
            starts.append((int(f["a"]), int(f["b"])))
    assert [(c["eff_batch"], c["n_decode"]) for c in fx] == starts
    for c in fx:
        assert sum(r[2] for r in c["rows"]) == c["eff_batch"]
        assert sum(r[4] for r in c["rows"]) == c["n_decode"]


def test_reference_arm_does_not_load_the_product(tmp_path):
    """bench.py's CPU legs import only oracle/: a process running them has no libdeserve_b200.so
    mapped (the reference arm measures the reference's CPU path, nothing of ours)."""
    code = (
        "import sys, os; sys.path.insert(0, %r); import bench\n"
        "circs = bench.systematic_sample(761, 3)\n"
        "import oracle\n"
        "fx = oracle.load_schedule_fixture(bench.SCHEDULE_FIXTURE)\n"
        "assert len(fx) == 761 and circs == sorted(set(circs))\n"
        "maps = open('/proc/self/maps').read()\n"
        "assert 'libdeserve_b200' not in maps, 'product library loaded'\n"
        "assert 'paper_2501_14784_b200' not in sys.modules\n"
        "print('ok')\n" % ROOT)
    r = subprocess.run([sys.executable, "-c", code], capture_output=True, text=True, timeout=120)
    assert r.returncode == 0 and r.stdout.strip() == "ok", r.stderr[-500:]


def test_pipesim_timing_runs_on_one_core():
    r = subprocess.run([sys.executable, os.path.join(ROOT, "oracle", "time_pipesim.py"),
                        os.path.join(CONFIGS, "llama8b_1stage.json"), "1"],
                       capture_output=True, text=True, timeout=120)
    assert r.returncode == 0, r.stderr[-500:]
    d = json.loads(r.stdout.strip().splitlines()[-1])
    assert d["cores"] == 1 and d["simulated_output_tokens"] == 68699 and d["wall_s"] > 0


@pytest.mark.parametrize("var", ["DS_SKIP", "DS_ATTN_SKIP", "DS_GEMM_NOFINISH"])
def test_bench_refuses_invalidating_switches(var):
    env = dict(os.environ, **{var: "1"})
    r = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--steps", "1"],
                       capture_output=True, text=True, timeout=120, env=env)
    assert r.returncode != 0 and var in r.stderr


@pytest.mark.parametrize("n", [2, 4, 8])
def test_multi_gpu_config_is_shared_and_product_free(n):
    """The N>1 arm's `config` comes from the config document alone (bench_multi.arm_config), so
    the reference arm under torchrun prints the identical dict without loading the product."""
    code = (
        "import sys, json; sys.path.insert(0, %r); import bench_multi\n"
        "c = bench_multi.arm_config(%d)\n"
        "assert 'paper_2501_14784_b200' not in sys.modules\n"
        "print(json.dumps(c))\n" % (ROOT, n))
    r = subprocess.run([sys.executable, "-c", code], capture_output=True, text=True, timeout=120)
    assert r.returncode == 0, r.stderr[-500:]
    c = json.loads(r.stdout.strip().splitlines()[-1])
    assert c["parallelism"] == f"pp{n}" and f"{n}-stage pipeline on {n}xB200" in c["workload"]
    assert "32 microbatches" in c["workload"] and "KV swap on" in c["workload"]
    assert set(c) == {"workload", "parallelism", "hops"}  # no run-dependent fields


@pytest.mark.parametrize("run,lo", [("r02_70b_8stage_4gpu", 0.9), ("r02_8b_4stage_swap_pin", 0.95),
                                    ("r02_70b_4stage_swap_pin", 0.5)])
def test_pipeline_roofline_of_committed_runs(run, lo):
    """SURVEY.md 8(d) pipeline fraction of the committed multi-stage B200 runs
    (tools/pipeline_roofline.py): every last-stage compute in the window maps onto its schedule
    circuit (checked), and the windowed output throughput sits below the roofline bound."""
    sys.path.insert(0, os.path.join(ROOT, "tools"))
    import pipeline_roofline
    r = pipeline_roofline.pipeline_roofline(os.path.join(ROOT, "profiles", run))
    assert r["circuits_in_window"] > 1000
    assert lo <= r["pipeline_fraction"] <= 1.0
    committed = json.load(open(os.path.join(ROOT, "profiles", run, "pipeline_roofline.json")))
    assert committed["pipeline_fraction"] == r["pipeline_fraction"]


def test_pipeline_roofline_of_the_n4_bench_run():
    """The same for the committed N=4 bench run (one process per GPU over NCCL; its config is
    bench_multi.pipeline_config(4), BASELINE configs[2] as written)."""
    sys.path.insert(0, os.path.join(ROOT, "tools"))
    import bench_multi
    import pipeline_roofline
    d = os.path.join(ROOT, "profiles", "r02_bench_n4")
    r = pipeline_roofline.pipeline_roofline(d, json.dumps(bench_multi.pipeline_config(4)))
    assert 0.9 <= r["pipeline_fraction"] <= 1.0 and r["stages"] == 4
    assert json.load(open(os.path.join(d, "pipeline_roofline.json")))["pipeline_fraction"] == r["pipeline_fraction"]


def test_committed_n1_bench_line_is_self_consistent():
    """profiles/r02_bench_n1_latest.json (the default `python bench.py` on a B200): value =
    decode tokens of the offline batch / ms_per_step; roofline.frac = achieved / peak with achieved
    = algorithmic bytes per launch / average launch time; stage_roofline recomputed here from the
    schedule equals the line's, and its frac = t_roof / ms_per_step."""
    sys.path.insert(0, ROOT)
    import bench
    d = json.load(open(os.path.join(ROOT, "profiles", "r02_bench_n1_latest.json")))
    assert d["report"]["output_tokens"] == d["workload_detail"]["tokens_per_step"] == 68699
    assert abs(d["value"] - 68699 / (d["ms_per_step"] / 1e3)) < 0.01 * d["value"] / 100
    rf = d["roofline"]
    ach = rf["algorithmic_bytes_per_launch"] / (rf["avg_launch_ms"] / 1e3) / 1e9
    assert abs(ach - rf["achieved"]) < 0.01 and abs(rf["achieved"] / rf["peak"] - rf["frac"]) < 1e-4
    if os.path.exists(os.path.join(ROOT, "MEASURED_PEAKS.json")):
        sr = bench.stage_roofline(open(os.path.join(CONFIGS, "llama8b_1stage.json")).read())
        assert sr["t_roof_s_per_step"] == d["stage_roofline"]["t_roof_s_per_step"]
    assert abs(d["stage_roofline"]["t_roof_s_per_step"] / (d["ms_per_step"] / 1e3)
               - d["stage_roofline"]["frac"]) < 1e-4
    assert d["e2e"]["value"] > 0.99 * d["value"] and d["gpu_launches"] > 0


def test_roofline_traffic_and_70b_summary_come_from_the_committed_captures():
    """The bench line's roofline.traffic is the DRAM read + write of the committed ncu --set full
    capture it names; profiles/r02_70b_shapes/summary.json is tools/summarize_cal70.py applied
    to the committed launch list."""
    import csv
    d = json.load(open(os.path.join(ROOT, "profiles", "r02_bench_n1_latest.json")))
    rows = list(csv.reader(open(os.path.join(ROOT, "profiles", "r02_ncu_full_gemm_gate_up.csv"))))
    h, units, v = rows[0], rows[1], rows[2]
    mb = {"Mbyte": 1e6, "Kbyte": 1e3, "byte": 1.0, "Gbyte": 1e9}
    rd = float(v[h.index("dram__bytes_read.sum")]) * mb[units[h.index("dram__bytes_read.sum")]]
    wr = float(v[h.index("dram__bytes_write.sum")]) * mb[units[h.index("dram__bytes_write.sum")]]
    assert abs(rd + wr - d["roofline"]["traffic"]) < 1.0
    s70 = os.path.join(ROOT, "profiles", "r02_70b_shapes")
    r = subprocess.run([sys.executable, os.path.join(ROOT, "tools", "summarize_cal70.py"),
                        os.path.join(s70, "cal70_launches.csv"), os.path.join(ROOT, "MEASURED_PEAKS.json")],
                       capture_output=True, text=True, timeout=120, cwd=ROOT)
    assert r.returncode == 0, r.stderr[-300:]
    got, want = json.loads(r.stdout), json.load(open(os.path.join(s70, "summary.json")))
    assert got["configs"] == want["configs"]
    dec = {c["T"]: c["kinds"]["attention_decode"]["alg_frac_of_hbm"] for c in got["configs"] if c["T"] < 1000}
    assert dec[49] >= 0.7 and dec[256] >= 0.7  # the north-star decode-attention target at 70B
