"""Per-step times of the bench's e2e leg (cfg3 through apply_filter_host, pinned host buffers)."""
import sys, time
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import numpy as np
import torch
import paper_2203_10213_b200 as vk

n = 1024
k = vk.gaussian_kernel(1.5)
rz = 3
plane_b = n * n * 2
src = vk.synthetic_device((n, n, n), vk.DataFormat.UINT16, seed=7)
pin_in = torch.empty((n + 2 * rz) * plane_b, dtype=torch.uint8, pin_memory=True)
pin_out = torch.empty((n + 2 * rz) * plane_b, dtype=torch.uint8, pin_memory=True)
pin_in[rz * plane_b:(rz + n) * plane_b].copy_(src.data.array)
host_in = pin_in.numpy().view(np.uint16).reshape(n + 2 * rz, n, n)
host_out = pin_out.numpy().view(np.uint16).reshape(n + 2 * rz, n, n)
host_in[:rz] = host_in[rz]
host_in[n + rz:] = host_in[n + rz - 1]
hl, hh = np.ascontiguousarray(host_in[:rz]), np.ascontiguousarray(host_in[n + rz:])
for label, kw in (("pinned halos", dict(halo_lo=host_in[:rz], halo_hi=host_in[n + rz:])),
                  ("copied halos", dict(halo_lo=hl, halo_hi=hh))):
    for path in ("auto", "dense"):
        vk.set_execution_policy(vk.ExecutionPolicy(filter_path=path))
        ts = []
        for i in range(8):
            torch.cuda.synchronize()
            t = time.perf_counter()
            vk.apply_filter_host(host_in[rz:n + rz], k, "clamp", out=host_out[rz:n + rz], z_offset=0,
                                 global_nz=n, **kw)
            torch.cuda.synchronize()
            ts.append((time.perf_counter() - t) * 1e3)
        print(f"[{label} {path}] " + " ".join(f"{t:.1f}" for t in ts), flush=True)
vk.set_execution_policy(vk.ExecutionPolicy())
