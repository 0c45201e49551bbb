"""Summarise an ncu launch list (`ncu --metrics gpu__time_duration.sum --csv --log-file X.csv ...`):
per kernel: launches, total and per-launch time, share of all kernel time.

  python tools/launch_list.py X.csv "<command it profiled>" > profiles/<round>_launches_bench.txt
"""
import csv
import sys
from collections import defaultdict

rows = list(csv.reader(open(sys.argv[1])))
hdr = next(i for i, r in enumerate(rows) if "Kernel Name" in r and "Metric Value" in r)
h = rows[hdr]
ix = {k: i for i, k in enumerate(h)}
tot = defaultdict(float)
cnt = defaultdict(int)
for r in rows[hdr + 1:]:
    if len(r) < len(h) or r[ix["Metric Name"]] != "gpu__time_duration.sum":
        continue
    v = float(r[ix["Metric Value"]].replace(",", ""))
    unit = r[ix["Metric Unit"]]
    ms = v * {"ns": 1e-6, "nsecond": 1e-6, "us": 1e-3, "usecond": 1e-3, "ms": 1.0, "msecond": 1.0,
              "s": 1e3, "second": 1e3}[unit]
    name = r[ix["Kernel Name"]]
    tot[name] += ms
    cnt[name] += 1
all_ms = sum(tot.values())
print(f"# ncu launch list of `{sys.argv[2] if len(sys.argv) > 2 else '?'}`")
print("# gpu__time_duration.sum, --clock-control none; cold-cache serialized launches: compare SHARES\n")
for name, ms in sorted(tot.items(), key=lambda kv: -kv[1]):
    print(f"{cnt[name]:4d} launches {ms:10.3f} ms total {ms / cnt[name]:10.3f} ms/launch {100 * ms / all_ms:5.1f}%  {name[:110]}")
