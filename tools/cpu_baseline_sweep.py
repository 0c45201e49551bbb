"""Rate of the reference's own apply_filter (baseline/_ref) against the sample
shape used by bench.py's CPU baseline: planes (= 4 x threads and multiples)
and rows per plane, full 1024-cell rows, u16 gaussian 7^3 Clamp.

  python tools/cpu_baseline_sweep.py [planes ...]  > profiles/r02_cpu_baseline_sweep.txt
"""

import os
import sys
import time
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT / "baseline" / "_ref"))
import vkt  # noqa: E402  (the unmodified reference)

threads = len(os.sched_getaffinity(0))
vkt.set_execution_policy(vkt.ExecutionPolicy(worker_count=0))
k = vkt.gaussian_kernel(1.5)
rng = np.random.default_rng(7)
plane_list = [int(a) for a in sys.argv[1:]] or [4 * threads, 8 * threads, 16 * threads]
print(f"# reference vkt.apply_filter, {threads} host threads (effective_workers={vkt.effective_workers()})")
print("planes rows slabs slab_thickness voxels seconds gvox_s")
for planes in plane_list:
    for rows in (256, 1024):
        v = vkt.StructuredVolume((1024, rows, planes), vkt.DataFormat.UINT16)
        v.array()[...] = rng.integers(0, 65536, size=v.array().shape, dtype=np.uint16)
        slabs = vkt.execution.slab_ranges(planes)
        t0 = time.perf_counter()
        vkt.apply_filter(v, k)
        dt = time.perf_counter() - t0
        n = 1024 * rows * planes
        print(f"{planes} {rows} {len(slabs)} {slabs[0][1] - slabs[0][0]} {n} {dt:.2f} {n / dt / 1e9:.6f}", flush=True)
