"""Summarise an ncu report: key throughput metrics, stall reasons, hottest SASS."""
import csv
import subprocess
import sys
from collections import Counter

rep = sys.argv[1]
raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(raw.splitlines()))
hdr, vals = rows[0], rows[2]
want = ['gpu__time_duration.sum', 'dram__bytes_read.sum', 'dram__bytes_write.sum',
        'smsp__issue_active.avg.pct_of_peak_sustained_active', 'sm__warps_active.avg.pct_of_peak_sustained_active',
        'sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active', 'launch__registers_per_thread',
        'launch__occupancy_limit_registers', 'launch__occupancy_limit_shared_mem', 'smsp__inst_executed.sum',
        'launch__grid_size', 'dram__throughput.avg.pct_of_peak_sustained_elapsed', 'lts__t_sector_hit_rate.pct']
for h, v in zip(hdr, vals):
    if h in want:
        print(f"{h:70s} {v}")
for h, v in zip(hdr, vals):
    if 'issue_stalled' in h and 'per_issue_active' in h and float(v or 0) > 0.05:
        print(f"  stall {h.split('stalled_')[1].split('_per')[0]:24s} {float(v):.3f}")
if len(sys.argv) > 2:
    src = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"],
                         capture_output=True, text=True).stdout
    srows = list(csv.reader(src.splitlines()))
    h2 = srows[1]
    ix = {h: i for i, h in enumerate(h2)}
    data = srows[2:]
    k = "Warp Stall Sampling (All Samples)"
    tot = sum(float(r[ix[k]] or 0) for r in data) or 1
    c = Counter()
    for r in data:
        t = r[ix["Source"]].split()
        if not t:
            continue
        op = t[1] if t[0].startswith('@') else t[0]
        c[op.split('.')[0]] += float(r[ix[k]] or 0)
    print("stall samples by opcode:", ", ".join(f"{op} {100 * v / tot:.1f}%" for op, v in c.most_common(10)))
    for r in sorted(data, key=lambda r: -float(r[ix[k]] or 0))[:int(sys.argv[2])]:
        print(f"  {float(r[ix[k]]) / tot * 100:5.1f}% {r[ix['Address']][-5:]} x{r[ix['Instructions Executed']]:>10s}  {r[ix['Source']][:75]}")
