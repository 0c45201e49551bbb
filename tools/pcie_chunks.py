"""Chunked copy experiments: which ingredient slows H2D inside the host pipeline."""
import sys
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import torch
import paper_2203_10213_b200 as vk

C = 122 << 20
N = 16
pin = torch.empty(N * C, dtype=torch.uint8, pin_memory=True)
pout = torch.empty(N * C, dtype=torch.uint8, pin_memory=True)
din = [torch.empty(C, dtype=torch.uint8, device="cuda") for _ in range(4)]
dout = [torch.empty(C, dtype=torch.uint8, device="cuda") for _ in range(4)]
sa, sb, sc = torch.cuda.Stream(), torch.cuda.Stream(), torch.cuda.Stream()
src = vk.synthetic_device((1024, 1024, 64), vk.DataFormat.UINT16, seed=7)
dst = vk.StructuredVolume(src.dims, src.format)
k = vk.gaussian_kernel(1.5)


def run(h2d=True, d2h=True, d2d=False, kern=False):
    torch.cuda.synchronize()
    e = [torch.cuda.Event(enable_timing=True) for _ in range(6)]
    e[0].record(sa); e[2].record(sb); e[4].record(sc)
    for i in range(N):
        if h2d:
            with torch.cuda.stream(sa):
                if d2d:
                    din[i % 4][: 12 << 20].copy_(din[(i + 3) % 4][-(12 << 20):], non_blocking=True)
                din[i % 4].copy_(pin[i * C:(i + 1) * C], non_blocking=True)
        if d2h:
            with torch.cuda.stream(sb):
                pout[i * C:(i + 1) * C].copy_(dout[i % 4], non_blocking=True)
        if kern:
            with torch.cuda.stream(sc):
                vk.ApplyFilter(dst, src, k)
    e[1].record(sa); e[3].record(sb); e[5].record(sc)
    torch.cuda.synchronize()
    ta, tb, tc = e[0].elapsed_time(e[1]), e[2].elapsed_time(e[3]), e[4].elapsed_time(e[5])
    gb = N * C / 1e6
    return f"H2D {ta:6.1f} ms ({gb / ta:5.1f} GB/s)  D2H {tb:6.1f} ms ({gb / tb:5.1f} GB/s)  kern {tc:6.1f} ms"


for rep in range(2):
    print("h2d only         ", run(d2h=False))
    print("d2h only         ", run(h2d=False))
    print("h2d||d2h         ", run())
    print("h2d+d2d||d2h     ", run(d2d=True))
    print("h2d||d2h||kernel ", run(kern=True))
    print("h2d+d2d||d2h||k  ", run(d2d=True, kern=True))
