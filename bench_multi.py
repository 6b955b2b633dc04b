"""N>1 leg of bench.py (see bench.py docstring). Placeholder until the multi-GPU path lands."""
import json
import os


def run_multi(args):
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return None
    return {"metric": "generated tokens/sec (whole pipeline) at injected inter-stage latency; roofline fraction",
            "value": None, "unit": "tokens/s", "n_gpus": args.gpus, "unavailable": "multi-GPU leg not built yet"}
