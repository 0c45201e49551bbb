#!/bin/bash
# f32 anisotropic kernels with x/y padding (or K = 3): the guarded cube path
# (Inf/NaN scan + tiled kernel) against the direct kernel, 512^3, Clamp.
# Roofline = slower of 8 B/voxel at HBM peak and kx*ky*kz FMAs at FP32 peak.
python - <<'PY'
import sys, torch
sys.path.insert(0, '.')
import numpy as np
import paper_2203_10213_b200 as vk
dims = (512, 512, 512)
nv = dims[0] * dims[1] * dims[2]
f = vk.DataFormat.FLOAT32
src = vk.synthetic_device(dims, f, seed=7)
dst = vk.StructuredVolume(src.dims, f, data=vk.DeviceBuffer(src.nbytes, zero=False))
st = torch.cuda.current_stream()
for kd in ((3, 1, 5), (5, 3, 5), (3, 3, 1), (1, 3, 3), (7, 5, 3), (9, 1, 1), (3, 3, 5)):
    n = kd[0] * kd[1] * kd[2]
    k = vk.Kernel(kd, np.full(n, 1.0 / n))
    t_roof = max(nv * 8 / 6541.5e9, nv * n / (148 * 128 * 1.965e9)) * 1e3
    row = []
    for path in ("auto", "direct"):
        vk.set_execution_policy(vk.ExecutionPolicy(filter_path=path))
        vk.ApplyFilter(dst, src, k, "clamp")
        best = 1e9
        for _ in range(5):
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record(st); vk.ApplyFilter(dst, src, k, "clamp"); b.record(st); b.synchronize()
            best = min(best, a.elapsed_time(b))
        row.append((path, vk.filter_path(dst, src, k), best))
    vk.set_execution_policy(vk.ExecutionPolicy())
    s = "  ".join(f"{p}[{q}] {t:.3f} ms ({t_roof / t:.3f} of roofline)" for p, q, t in row)
    print(f"f32 {dims} k={kd}: {s}  speed-up {row[1][2] / row[0][2]:.1f}x")
PY
