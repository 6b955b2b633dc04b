#!/usr/bin/env python3
"""Writes the row layout of every circuit of a config's schedule as a gzip JSON fixture
(configs/<name>.schedule.json.gz): [{"eff_batch", "n_decode", "rows": [[slot, pos, n_tok,
need_logits, is_decode, req_id], ...]}, ...]. The schedule is the reference Engine's decision
sequence (begin_circuit, /root/reference/proj/src/sim.cpp:386-407; our scheduler's trace is
byte-identical to the reference's, tests/test_integer_parity.py), so bench.py's reference arm can
time the CPU stage forward on the workload's real circuits without loading the product library.
tests/test_bench_cpu.py checks the fixture's (eff_batch, n_decode) against the reference's own
trace."""
import gzip
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    from paper_2501_14784_b200 import pipeline as pl
    name = sys.argv[1] if len(sys.argv) > 1 else "llama8b_1stage.json"
    cdir = os.path.join(ROOT, "configs")
    sc = pl.schedule_config(open(os.path.join(cdir, name)).read(), cdir)
    out = [{"eff_batch": c["eff_batch"], "n_decode": c["n_decode"], "rows": c["rows"]}
           for c in sc["circuits"]]
    path = os.path.join(cdir, name.replace(".json", ".schedule.json.gz"))
    with gzip.open(path, "wt") as f:
        json.dump(out, f, separators=(",", ":"))
    print(path, len(out), "circuits")


if __name__ == "__main__":
    main()
