"""One traced apply_filter_host run of cfg3 from pinned buffers (VKT_HOST_TRACE=1)."""
import os, sys, time
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import numpy as np
import torch
import paper_2203_10213_b200 as vk

n = 1024
chunk = int(sys.argv[1]) if len(sys.argv) > 1 else 0
nb = n * n * n * 2
pin = torch.empty(nb, dtype=torch.uint8, pin_memory=True)
pin2 = torch.empty(nb, dtype=torch.uint8, pin_memory=True)
src = vk.synthetic_device((n, n, n), vk.DataFormat.UINT16, seed=7)
pin.copy_(src.data.array)
hin = pin.numpy().view(np.uint16).reshape(n, n, n)
hout = pin2.numpy().view(np.uint16).reshape(n, n, n)
k = vk.gaussian_kernel(1.5)
vk.apply_filter_host(hin, k, out=hout, chunk_planes=chunk)
torch.cuda.synchronize()
t = time.perf_counter()
vk.apply_filter_host(hin, k, out=hout, chunk_planes=chunk)
print(f"untraced: {(time.perf_counter() - t) * 1e3:.1f} ms", flush=True)
os.environ["VKT_HOST_TRACE"] = "1"
t = time.perf_counter()
vk.apply_filter_host(hin, k, out=hout, chunk_planes=chunk)
print(f"traced: {(time.perf_counter() - t) * 1e3:.1f} ms", flush=True)
