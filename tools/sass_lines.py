"""Static SASS instructions per source line for one kernel of a -lineinfo cubin.

  nvcc ... -lineinfo -cubin -o X.cubin file.cu
  python tools/sass_lines.py X.cubin MANGLED_NAME_SUBSTR [top]
"""
import collections
import re
import subprocess
import sys

txt = subprocess.run(["nvdisasm", "-g", "-c", sys.argv[1]], capture_output=True, text=True).stdout
marker = "//--------------------- .text."
parts = txt.split(marker)
sec = next(p for p in parts[1:] if p.startswith(sys.argv[2]) or sys.argv[2] in p.split("\n")[0])
cur = None
tot = collections.Counter()
ops = collections.defaultdict(collections.Counter)
for line in sec.split("\n"):
    m = re.search(r'//## File "([^"]+)", line (\d+)', line)
    if m:
        cur = (m.group(1).split("/")[-1], int(m.group(2)))
        continue
    m = re.match(r"\s+/\*[0-9a-f]+\*/\s+(@!?U?P\w+\s+)?([A-Z0-9_.]+)", line)
    if m and cur:
        tot[cur] += 1
        ops[cur][m.group(2).split(".")[0]] += 1
print("total", sum(tot.values()))
for k, v in sorted(tot.items(), key=lambda kv: -kv[1])[: int(sys.argv[3]) if len(sys.argv) > 3 else 40]:
    print(f"{v:5d}  {k[0]}:{k[1]:<5d} {dict(ops[k].most_common(5))}")
