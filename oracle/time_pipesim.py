#!/usr/bin/env python3
"""TEST INFRASTRUCTURE / CPU BASELINE ONLY: times the reference CPU path itself -- pipesim run()
(/root/reference/proj/src/sim.cpp:534-595, compiled unmodified into oracle/_ref) -- on a config,
single-threaded by design, pinned to one core. The config's node calibration is the
measured B200 CSV (configs/cal_b200_*.csv), so run() predicts the GPU pipeline's throughput from
the reference's own event engine. Prints one JSON object: simulated output tok/s, wall seconds,
events/s."""
import json
import os
import sys
import time

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.dirname(HERE))


def main():
    import oracle
    cfg = sys.argv[1]
    reps = int(sys.argv[2]) if len(sys.argv) > 2 else 3
    try:
        os.sched_setaffinity(0, {min(os.sched_getaffinity(0))})
    except (AttributeError, OSError):
        pass
    ref = oracle.Ref()
    txt, cdir = open(cfg).read(), os.path.dirname(os.path.abspath(cfg))
    walls, rep = [], None
    for _ in range(reps):
        t0 = time.perf_counter()
        rep = ref.sim_config(txt, cdir)
        walls.append(time.perf_counter() - t0)
    trace = os.path.join("/tmp", f"pipesim_{os.getpid()}.trace")
    ref.sim_config(txt, cdir, trace_path=trace)
    n_ev, makespan = 0, 0
    for line in open(trace):
        n_ev += 1
        if "kind=ComputeEnd" in line:
            makespan = max(makespan, int(line.split()[0][2:]))
    os.remove(trace)
    w = sorted(walls)[len(walls) // 2]
    print(json.dumps({"impl": "pipesim run() (oracle/_ref, unmodified reference sources)",
                      "cores": 1, "wall_s": round(w, 6), "events": n_ev,
                      "events_per_s": round(n_ev / w, 1),
                      "simulated_output_tokens_per_s": rep["output_throughput"],
                      "simulated_output_tokens": rep["output_tokens"],
                      "window_s": rep["wall_time_s"],
                      # offline batch (BASELINE configs[1]): N_O / makespan
                      "makespan_s": makespan / 1e6,
                      "simulated_tokens_per_s_makespan": rep["output_tokens"] * 1e6 / max(makespan, 1)}))


if __name__ == "__main__":
    main()
