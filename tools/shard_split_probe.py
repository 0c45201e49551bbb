"""Cost of the sharded launch split on one GPU: per-rank slab (1024^2 x n, u16,
7^3) with halo buffers, as one launch vs interior + two boundary launches."""
import sys
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import torch
import paper_2203_10213_b200 as vk
from paper_2203_10213_b200.filters import make_args, launch

k = vk.gaussian_kernel(1.5)
fmt = vk.DataFormat.UINT16
rz = 3
for n in (512, 256, 128, 64):
    src = vk.synthetic_device((1024, 1024, n), fmt, seed=7)
    dst = vk.StructuredVolume(src.dims, fmt, data=vk.DeviceBuffer(src.nbytes, zero=False))
    pb = 1024 * 1024 * 2
    lo = torch.empty(rz * pb, dtype=torch.uint8, device="cuda")
    hi = torch.empty(rz * pb, dtype=torch.uint8, device="cuda")
    common = dict(dims=(1024, 1024, n), fmt=fmt, mapping=(0.0, 1.0), kernel=k, mode=vk.AddressMode.CLAMP,
                  z_offset=1024, global_nz=4096, halo_lo=lo.data_ptr(), halo_hi=hi.data_ptr())
    s = torch.cuda.current_stream()
    def run(split):
        rngs = ((rz, n - rz), (0, rz), (n - rz, n)) if split else ((0, n),)
        for b, e in rngs:
            a, _keep = make_args(dst.data_ptr(), src.data_ptr(), **common, out_z_begin=b, out_z_end=e)
            launch(a, int(s.cuda_stream))
    for split in (False, True):
        for _ in range(2):
            run(split)
        ts = []
        for _ in range(5):
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(s); run(split); e1.record(s); e1.synchronize(); ts.append(e0.elapsed_time(e1))
        print(f"n={n:4d} {'interior+2 boundary' if split else 'one launch         '}: {min(ts):.3f} ms")
