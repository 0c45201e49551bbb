#!/bin/bash
# the generic direct kernel on shapes the tiled kernel does not take (anisotropic, K = 9)
python - <<'PY'
import sys, torch
sys.path.insert(0, '.')
import numpy as np
import paper_2203_10213_b200 as vk
for fmt, dims, kd in (("u8", (512, 512, 512), (3, 1, 5)), ("f32", (512, 512, 512), (5, 5, 1)), ("u16", (512, 512, 512), (9, 9, 9)), ("f32", (512, 512, 512), (7, 7, 7))):
    f = vk.DataFormat.parse(fmt)
    src = vk.synthetic_device(dims, f, seed=7)
    dst = vk.StructuredVolume(src.dims, f, data=vk.DeviceBuffer(src.nbytes, zero=False))
    n = kd[0] * kd[1] * kd[2]
    k = vk.Kernel(kd, np.full(n, 1.0 / n))
    st = torch.cuda.current_stream()
    vk.ApplyFilter(dst, src, k, "clamp")
    best = 1e9
    for _ in range(3):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(st); vk.ApplyFilter(dst, src, k, "clamp"); b.record(st); b.synchronize()
        best = min(best, a.elapsed_time(b))
    nv = dims[0] * dims[1] * dims[2]
    fr = nv * n / (148 * 128 * 1.965e9) / (best / 1e3)
    print(f"{fmt} {dims} k={kd} path={vk.filter_path(dst, src, k)}: {best:.3f} ms = {nv / best / 1e6:.1f} GVox/s, FP32 roofline fraction {fr:.3f}")
PY
