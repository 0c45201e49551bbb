"""Executed-instruction mix by opcode from an ncu report's source page."""
import csv, subprocess, sys
from collections import Counter
src = subprocess.run(["ncu", "-i", sys.argv[1], "--page", "source", "--csv", "--print-source", "sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(src.splitlines()))
h = rows[1]; ix = {k: i for i, k in enumerate(h)}
c = Counter()
for r in rows[2:]:
    t = r[ix["Source"]].split()
    if not t:
        continue
    op = t[1] if t[0].startswith('@') else t[0]
    c[op] += int(r[ix["Instructions Executed"]] or 0)
tot = sum(c.values())
print(f"total warp instructions {tot:.4g}")
for op, n in c.most_common(int(sys.argv[2]) if len(sys.argv) > 2 else 25):
    print(f"  {op:28s} {n:14d} {100 * n / tot:5.1f}%")
