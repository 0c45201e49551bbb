"""Registers / spills per kernel: python tools/ptxas_regs.py paper_2203_10213_b200/csrc/filter_tma_u16.cu"""
import re, subprocess, sys
cmd = ["nvcc", "-gencode", "arch=compute_100a,code=sm_100a", "-O3", "-std=c++17", "--expt-relaxed-constexpr",
       "-I", "include", "-Xptxas", "-v", "-cubin", "-o", "/dev/null", sys.argv[1]] + sys.argv[2:]
err = subprocess.run(cmd, capture_output=True, text=True).stderr
name = None
for line in err.splitlines():
    m = re.search(r"Compiling entry function '(\S+)'", line)
    if m:
        dm = subprocess.run(["c++filt"], input=m.group(1), capture_output=True, text=True).stdout.strip()
        name = re.sub(r"\(CUtensorMap_st.*", "", dm).replace("vkt::", "")
    m = re.search(r"(\d+) bytes spill stores", line)
    if m and name:
        spill = m.group(1)
    m = re.search(r"Used (\d+) registers", line)
    if m and name:
        print(f"{m.group(1):>4} regs  spill {spill:>4}  {name}")
        name = None
