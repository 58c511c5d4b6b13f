"""Aggregate an ncu --csv launch list with several metrics per kernel name (mean per launch).
Usage: python tools/ncu_agg.py <launches.csv>"""
import collections
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
st = next(i for i, r in enumerate(rows) if r and r[0] == "ID")
h = rows[st]
ix = {k: j for j, k in enumerate(h)}
d = collections.defaultdict(dict)
for r in rows[st + 1:]:
    if len(r) < len(h):
        continue
    d[(r[ix["ID"]], r[ix["Kernel Name"]])][r[ix["Metric Name"]]] = float(r[ix["Metric Value"]].replace(",", ""))
agg = collections.defaultdict(lambda: collections.defaultdict(float))
cnt = collections.Counter()
for (i, k), m in d.items():
    cnt[k] += 1
    for mk, v in m.items():
        agg[k][mk] += v
for k in sorted(agg, key=lambda k: -agg[k]["gpu__time_duration.sum"]):
    n = cnt[k]
    print(n, {mk.split(".")[0].replace("sm__pipe_tensor_subpipe_", ""): round(v / n / (1e3 if "time" in mk else (1e6 if "bytes" in mk else 1)), 2)
              for mk, v in agg[k].items()}, k[:120])
