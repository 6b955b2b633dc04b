"""Summaries of ncu outputs for profiles/: launch-list shares by kernel, and key counters of
full captures (duration, DRAM bytes, throughput %, tensor-pipe %, occupancy)."""
import csv
import io
import subprocess
import sys
from collections import defaultdict


def launch_shares(path):
    rows = [l for l in open(path) if l.startswith('"')]
    rd = csv.DictReader(io.StringIO("".join(rows)))
    tot = defaultdict(float)
    cnt = defaultdict(int)
    for r in rd:
        if r.get("Metric Name") != "gpu__time_duration.sum":
            continue
        k = r["Kernel Name"].split("(")[0].replace("void ", "")
        v = float(r["Metric Value"].replace(",", ""))
        unit = r.get("Metric Unit", "ns")
        v = v / 1e3 if unit == "ns" else (v * 1e3 if unit == "ms" else v)  # -> us
        tot[k] += v
        cnt[k] += 1
    s = sum(tot.values())
    out = ["kernel,launches,total_us,share"]
    for k, v in sorted(tot.items(), key=lambda x: -x[1]):
        out.append(f"{k},{cnt[k]},{v:.1f},{v / s:.4f}")
    return "\n".join(out)


def full(path):
    raw = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True,
                         text=True).stdout
    rd = list(csv.reader(io.StringIO(raw)))
    h = rd[0]
    want = ["Kernel Name", "gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
            "gpu__compute_memory_throughput.avg.pct_of_peak_sustained_elapsed",
            "dram__throughput.avg.pct_of_peak_sustained_elapsed",
            "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active",
            "sm__throughput.avg.pct_of_peak_sustained_elapsed", "launch__grid_size",
            "launch__registers_per_thread", "sm__warps_active.avg.pct_of_peak_sustained_active",
            "lts__t_sector_hit_rate.pct"]
    idx = [(w, h.index(w)) for w in want if w in h]
    out = io.StringIO()
    wr = csv.writer(out, lineterminator="\n")
    wr.writerow([w for w, _ in idx])
    wr.writerow([rd[1][i] for _, i in idx])
    for r in rd[2:]:
        wr.writerow([r[i].split("(")[0] for _, i in idx])
    return out.getvalue().rstrip("\n")


if __name__ == "__main__":
    kind, path = sys.argv[1], sys.argv[2]
    print(launch_shares(path) if kind == "launches" else full(path))
