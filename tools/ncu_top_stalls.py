"""Hottest SASS instructions by stall samples, with their top reasons.

  python tools/ncu_top_stalls.py REPORT.ncu-rep [N]
"""
import csv
import subprocess
import sys

rep = sys.argv[1]
n = int(sys.argv[2]) if len(sys.argv) > 2 else 40
src = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(src.splitlines()))
h = rows[1]
ix = {k: i for i, k in enumerate(h)}
reasons = [k for k in h if k.startswith("stall_") and "Not Issued" not in k]
data = []
for r in rows[2:]:
    try:
        st = {k: float(r[ix[k]] or 0) for k in reasons}
        data.append((sum(st.values()), r[ix["Address"]], r[ix["Source"]], st, int(r[ix["Instructions Executed"]] or 0)))
    except (ValueError, IndexError):
        pass
T = sum(d[0] for d in data)
for t, a, s, st, ne in sorted(data, key=lambda d: -d[0])[:n]:
    main = sorted(st.items(), key=lambda kv: -kv[1])[:3]
    print(f"{100 * t / T:5.2f}% {a[-5:]} {ne:>10} {s[:62]:62s} " + " ".join(f"{k[6:]}:{100 * v / T:.2f}" for k, v in main))
