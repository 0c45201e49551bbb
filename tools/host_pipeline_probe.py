"""Diagnose the host-buffer pipeline: PCIe rates and apply_filter_host vs chunk size."""
import sys, time
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import numpy as np
import torch
import paper_2203_10213_b200 as vk

n = 1024
nb = n * n * n * 2
pin = torch.empty(nb, dtype=torch.uint8, pin_memory=True)
pin2 = torch.empty(nb, dtype=torch.uint8, pin_memory=True)
d = torch.empty(nb, dtype=torch.uint8, device="cuda")
for name, fn in (("H2D", lambda: d.copy_(pin, non_blocking=True)), ("D2H", lambda: pin2.copy_(d, non_blocking=True))):
    fn(); torch.cuda.synchronize()
    t = time.perf_counter(); fn(); torch.cuda.synchronize(); dt = time.perf_counter() - t
    print(f"{name} pinned 2 GiB: {dt*1e3:.1f} ms = {nb/dt/1e9:.1f} GB/s")
s2 = torch.cuda.Stream()
torch.cuda.synchronize(); t = time.perf_counter()
with torch.cuda.stream(s2):
    pin2.copy_(d, non_blocking=True)
d.copy_(pin, non_blocking=True)
torch.cuda.synchronize(); dt = time.perf_counter() - t
print(f"H2D||D2H pinned 2 GiB each: {dt*1e3:.1f} ms")
src = vk.synthetic_device((n, n, n), vk.DataFormat.UINT16, seed=7)
pin.copy_(src.data.array)
hin = pin.numpy().view(np.uint16).reshape(n, n, n)
hout = pin2.numpy().view(np.uint16).reshape(n, n, n)
k = vk.gaussian_kernel(1.5)
for path in ("auto", "dense"):
    vk.set_execution_policy(vk.ExecutionPolicy(filter_path=path))
    for chunk in (0, 16, 32, 64, 128, 256):
        vk.apply_filter_host(hin, k, out=hout, chunk_planes=chunk)
        t = time.perf_counter()
        for _ in range(3):
            vk.apply_filter_host(hin, k, out=hout, chunk_planes=chunk)
        dt = (time.perf_counter() - t) / 3
        print(f"[{path}] apply_filter_host chunk={chunk or 'auto'}: {dt*1e3:.1f} ms")
vk.set_execution_policy(vk.ExecutionPolicy())
pg_in = np.array(hin)  # pageable
pg_out = np.empty_like(pg_in)
vk.apply_filter_host(pg_in, k, out=pg_out, chunk_planes=128)
t = time.perf_counter(); vk.apply_filter_host(pg_in, k, out=pg_out, chunk_planes=128); dt = time.perf_counter() - t
print(f"apply_filter_host pageable chunk=128: {dt*1e3:.1f} ms")
