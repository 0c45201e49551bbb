"""Stall samples split by warp role, guessed from per-instruction execution
counts (producer / consumer code executes different counts per launch).

  python tools/ncu_role_stalls.py REPORT.ncu-rep COUNT_A[,COUNT_B...]=NAME ...
"""
import csv, subprocess, sys, collections
rep = sys.argv[1]
groups = {}
for spec in sys.argv[2:]:
    counts, name = spec.split("=")
    for c in counts.split(","):
        groups[int(c)] = name
src = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(src.splitlines()))
h = rows[1]
ix = {k: i for i, k in enumerate(h)}
reasons = [k for k in h if k.startswith("stall_") and "Not Issued" not in k]
tot = collections.defaultdict(lambda: collections.Counter())
for r in rows[2:]:
    try:
        ne = int(r[ix["Instructions Executed"]] or 0)
        st = {k: float(r[ix[k]] or 0) for k in reasons}
    except (ValueError, IndexError):
        continue
    name = groups.get(ne, "other")
    tot[name].update(st)
    tot[name]["_inst"] += ne
T = sum(sum(v for k, v in c.items() if k != "_inst") for c in tot.values())
for name, c in sorted(tot.items()):
    s = sum(v for k, v in c.items() if k != "_inst")
    top = sorted(((k, v) for k, v in c.items() if k != "_inst"), key=lambda kv: -kv[1])[:6]
    print(f"{name:10s} {100 * s / T:5.1f}% of samples, {c['_inst']:.3e} warp-inst:  " +
          "  ".join(f"{k[6:]} {100 * v / T:.1f}" for k, v in top))
