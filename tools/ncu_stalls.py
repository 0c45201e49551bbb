"""Stall-reason totals and the instructions carrying each reason (ncu source page)."""
import csv, subprocess, sys
from collections import Counter, defaultdict
src = subprocess.run(["ncu", "-i", sys.argv[1], "--page", "source", "--csv", "--print-source", "sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(src.splitlines()))
h = rows[1]; ix = {k: i for i, k in enumerate(h)}
reasons = [k for k in h if k.startswith("stall_") and "Not Issued" not in k]
tot = Counter(); by = defaultdict(Counter)
for r in rows[2:]:
    t = r[ix["Source"]].split()
    if not t:
        continue
    op = (t[1] if t[0].startswith("@") else t[0]).split(".")[0]
    for k in reasons:
        v = float(r[ix[k]] or 0)
        tot[k] += v; by[k][op] += v
T = sum(tot.values())
for k, v in tot.most_common(10):
    print(f"{k:24s} {100 * v / T:5.1f}%   " + ", ".join(f"{o} {100 * n / T:.1f}" for o, n in by[k].most_common(5)))
