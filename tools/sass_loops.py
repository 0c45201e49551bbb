"""Hot loops (backward branches with many FFMA/FFMA2) of one kernel: python tools/sass_loops.py x.cubin NAME_SUBSTR [-v]"""
import re, subprocess, sys
from collections import Counter
txt = subprocess.run(["cuobjdump", "-sass", sys.argv[1]], capture_output=True, text=True).stdout
for f in txt.split("Function : ")[1:]:
    name = f.split("\n")[0]
    if sys.argv[2] not in name:
        continue
    ins = []
    for l in f.split("\n"):
        m = re.match(r"\s+/\*([0-9a-f]{4,})\*/\s+(.*?)\s*;", l)
        if m:
            ins.append((int(m.group(1), 16), m.group(2).strip()))
    print(name[:90])
    for a, t in ins:
        m = re.search(r"BRA.*?0x([0-9a-f]+)", t)
        if m and int(m.group(1), 16) < a:
            body = [x for x in ins if int(m.group(1), 16) <= x[0] <= a]
            c = Counter((x[1].split()[1] if x[1].startswith("@") else x[1].split()[0]) for x in body)
            if c["FFMA2"] + c["FFMA"] > 20:
                print(f"  loop {int(m.group(1), 16):x}-{a:x}: {len(body)} instr  " + ", ".join(f"{k} {v}" for k, v in c.most_common(8)))
                if "-v" in sys.argv:
                    for x in body:
                        if "FFMA" not in x[1]:
                            print(f"     {x[0]:5x} {x[1][:90]}")
