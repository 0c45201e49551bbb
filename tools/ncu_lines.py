"""Dynamic instruction counts per CUDA source line: an ncu report's SASS page
(instructions executed per address) joined with the -lineinfo line table of
the same kernel in the build's object file.

  python tools/ncu_lines.py REPORT.ncu-rep build/obj/filter_tma_u8.o MANGLED_SUBSTR [top]
"""
import collections
import csv
import os
import re
import subprocess
import sys
import tempfile

rep, obj, fn = sys.argv[1:4]
top = int(sys.argv[4]) if len(sys.argv) > 4 else 30
src = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(src.splitlines()))
h = rows[1]
ix = {k: i for i, k in enumerate(h)}
ex = []
for r in rows[2:]:
    try:
        ex.append((int(r[ix["Address"]], 16), int(r[ix["Instructions Executed"]] or 0), r[ix["Source"]]))
    except (ValueError, IndexError):
        pass
base = min(a for a, _, _ in ex)
with tempfile.TemporaryDirectory() as d:
    subprocess.run(["cuobjdump", "-xelf", "all", os.path.abspath(obj)], cwd=d, capture_output=True)
    cubins = [os.path.join(d, f) for f in os.listdir(d) if f.endswith(".cubin")]
    txt = "".join(subprocess.run(["nvdisasm", "-g", "-c", c], capture_output=True, text=True).stdout for c in cubins)
marker = "//--------------------- .text."
sec = next(p for p in txt.split(marker)[1:] if fn in p.split("\n")[0])
line_of = {}
cur = None
for line in sec.split("\n"):
    m = re.search(r'//## File "([^"]+)", line (\d+)', line)
    if m:
        cur = f"{m.group(1).split('/')[-1]}:{m.group(2)}"
        continue
    m = re.match(r"\s+/\*([0-9a-f]+)\*/\s+", line)
    if m and cur:
        line_of[int(m.group(1), 16)] = cur
tot = collections.Counter()
ops = collections.defaultdict(collections.Counter)
missing = 0
for a, n, s in ex:
    k = line_of.get(a - base)
    if k is None:
        missing += n
        continue
    tot[k] += n
    t = s.split()
    op = (t[1] if t and t[0].startswith("@") else t[0] if t else "?").split(".")[0]
    ops[k][op] += n
allv = sum(tot.values()) + missing
print(f"total {allv:.4g} warp instructions ({missing} unmapped)")
for k, v in tot.most_common(top):
    print(f"{100 * v / allv:5.1f}%  {k:28s} {dict(ops[k].most_common(4))}")
