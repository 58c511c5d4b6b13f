"""Summarise ncu outputs for profiles/ (run here, no GPU needed).

  python tools/ncu_summary.py launches <launches.csv>          -> per-kernel count / mean / share
  python tools/ncu_summary.py full <report.ncu-rep> [name]     -> key metrics per captured launch
"""
import collections
import csv
import json
import subprocess
import sys

KEYS = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "sm__pipe_tensor_subpipe_dmma_cycles_active.avg.pct_of_peak_sustained_active",
        "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed",
        "sm__inst_executed_pipe_fp64.avg.pct_of_peak_sustained_active",
        "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active",
        "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "lts__t_bytes.sum",
        "sm__warps_active.avg.pct_of_peak_sustained_active", "launch__registers_per_thread",
        "launch__grid_size", "launch__block_size", "launch__cluster_dim_y",
        "sm__throughput.avg.pct_of_peak_sustained_elapsed", "smsp__issue_active.avg.pct_of_peak_sustained_active"]


def launches(path):
    rows = list(csv.reader(open(path)))
    start = next(i for i, r in enumerate(rows) if r and r[0] == "ID")
    h = rows[start]
    idx = {k: j for j, k in enumerate(h)}
    d = collections.defaultdict(list)
    for r in rows[start + 1:]:
        if len(r) < len(h) or r[idx["Metric Name"]] != "gpu__time_duration.sum":
            continue
        name = r[idx["Kernel Name"]].split("(")[0]
        v = float(r[idx["Metric Value"]].replace(",", ""))
        unit = r[idx["Metric Unit"]]
        d[name].append(v * (1e-3 if unit == "nsecond" or unit == "ns" else (1.0 if unit in ("usecond", "us") else 1e3)))
    tot = sum(sum(v) for v in d.values())
    out = {k: {"launches": len(v), "mean_us": round(sum(v) / len(v), 2), "total_us": round(sum(v), 1),
               "share": round(sum(v) / tot, 4)} for k, v in sorted(d.items(), key=lambda kv: -sum(kv[1]))}
    return out


def full(path, name=None):
    raw = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(raw.splitlines()))
    h, units = rows[0], rows[1]
    scale = {"byte": 1.0, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "nsecond": 1e-3, "usecond": 1.0,
             "msecond": 1e3}
    out = []
    for r in rows[2:]:
        rec = {"kernel": r[h.index("Kernel Name")][:120]}
        if name and name not in rec["kernel"]:
            continue
        for k in KEYS:
            if k in h:
                j = h.index(k)
                v = r[j].replace(",", "")
                try:
                    f = float(v) * scale.get(units[j], 1.0)
                    key = k + (" [bytes]" if units[j] in ("byte", "Kbyte", "Mbyte", "Gbyte") else
                               " [us]" if units[j] in ("nsecond", "usecond", "msecond") else "")
                    rec[key] = f
                except ValueError:
                    rec[k] = v
        out.append(rec)
    return out


if __name__ == "__main__":
    mode, path = sys.argv[1], sys.argv[2]
    res = launches(path) if mode == "launches" else full(path, sys.argv[3] if len(sys.argv) > 3 else None)
    print(json.dumps(res, indent=1))
