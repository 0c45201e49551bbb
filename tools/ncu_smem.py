"""Shared-memory / pipe summary of ncu reports: python tools/ncu_smem.py a.ncu-rep [b.ncu-rep ...]"""
import csv
import subprocess
import sys

WANT = ['gpu__time_duration.sum', 'sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active',
        'smsp__issue_active.avg.pct_of_peak_sustained_active',
        'l1tex__data_pipe_lsu_wavefronts_mem_shared_op_ld.sum', 'l1tex__data_bank_conflicts_pipe_lsu_mem_shared_op_ld.sum',
        'l1tex__data_pipe_lsu_wavefronts_mem_shared_op_st.sum', 'l1tex__data_bank_conflicts_pipe_lsu_mem_shared_op_st.sum',
        'l1tex__data_pipe_lsu_wavefronts_mem_shared.sum.pct_of_peak_sustained_elapsed',
        'memory_l1_wavefronts_shared_ideal', 'launch__registers_per_thread', 'launch__shared_mem_per_block_dynamic',
        'smsp__inst_executed.sum', 'dram__bytes_read.sum', 'dram__bytes_write.sum', 'launch__grid_size']
for rep in sys.argv[1:]:
    raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(raw.splitlines()))
    h, v = rows[0], rows[2]
    print("==", rep)
    for a, b in zip(h, v):
        if a in WANT:
            print(f"  {a:80s} {b}")
    for a, b in zip(h, v):
        if 'issue_stalled' in a and 'per_issue_active' in a and float(b or 0) > 0.05:
            print(f"  stall {a.split('stalled_')[1].split('_per')[0]:24s} {float(b):.3f}")
