"""Static SASS opcode mix of one kernel in a cubin: python tools/sass_mix.py file.cubin NAME_SUBSTR"""
import collections, re, subprocess, sys
txt = subprocess.run(["cuobjdump", "-sass", sys.argv[1]], capture_output=True, text=True).stdout
for f in txt.split("Function : ")[1:]:
    name = f.split("\n")[0]
    if sys.argv[2] not in name:
        continue
    ops = collections.Counter()
    for line in f.split("\n"):
        m = re.match(r"\s+/\*[0-9a-f]+\*/\s+(@!?U?P\w+\s+)?([A-Z0-9_.]+)", line)
        if m:
            ops[m.group(2)] += 1
    print(name[:90])
    print(sum(ops.values()), ops.most_common(int(sys.argv[3]) if len(sys.argv) > 3 else 16))
