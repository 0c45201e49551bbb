"""Anisotropic kernels on the tiled path: time and roofline fraction.

Shapes (kx, ky, kz) from the round-1 verdict: (3,1,5), (5,3,5), (7,5,3),
(9,1,1), plus (1,1,9), (5,5,1), for u8 / u16 / f32 at 512^3, Clamp.  Roofline:
the slower of HBM (2 x bpc bytes / voxel at the measured peak) and FP32
(kx*ky*kz FMAs / voxel at 148 x 128 FMA/clk x 1965 MHz).

  python tools/aniso_rates.py [n]  -> one JSON line per case
"""
import json
import statistics
import sys
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))
import torch  # noqa: E402

import paper_2203_10213_b200 as vk  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 512
peaks = json.loads((ROOT / "MEASURED_PEAKS.json").read_text()) if (ROOT / "MEASURED_PEAKS.json").exists() else {}
HBM = float(peaks.get("hbm_gbs", 6545.3)) * 1e9
FMA = torch.cuda.get_device_properties(0).multi_processor_count * 128 * 1965e6
rng = np.random.default_rng(1)
for fmt in (vk.DataFormat.UINT8, vk.DataFormat.UINT16, vk.DataFormat.FLOAT32):
    src = vk.synthetic_device((n, n, n), fmt, seed=3)
    dst = vk.StructuredVolume(src.dims, fmt, data=vk.DeviceBuffer(src.nbytes, zero=False))
    for kd in ((3, 1, 5), (5, 3, 5), (7, 5, 3), (9, 1, 1), (1, 1, 9), (5, 5, 1)):
        w = rng.random(kd[::-1])
        w /= w.sum()
        kern = vk.Kernel(kd, w.reshape(-1))
        s = torch.cuda.current_stream()
        for _ in range(3):
            vk.ApplyFilter(dst, src, kern)
        ts = []
        for _ in range(10):
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record(s)
            vk.ApplyFilter(dst, src, kern)
            b.record(s)
            b.synchronize()
            ts.append(a.elapsed_time(b))
        ms = min(ts)
        nvox = n ** 3
        taps = kd[0] * kd[1] * kd[2]
        t_hbm = nvox * 2 * fmt.bytes_per_cell / HBM
        t_fma = nvox * taps / FMA
        bound = "fp32" if t_fma >= t_hbm else "hbm"
        print(json.dumps({"format": fmt.short_name, "kdims": kd, "n": n, "ms": round(ms, 4),
                          "gvox_s": round(nvox / ms / 1e6, 1), "path": vk.filter_path(dst, src, kern),
                          "bound": bound, "frac": round(max(t_hbm, t_fma) * 1e3 / ms, 3),
                          "median_ms": round(statistics.median(ts), 4)}), flush=True)
    del src, dst
    torch.cuda.empty_cache()
