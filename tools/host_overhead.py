"""Host-side cost of one ApplyFilter call vs the kernel's own duration.

  python tools/host_overhead.py [--n 256] [--fmt u8] [--k 3]

Prints: wall-clock us per call for a tiny (16^3) volume (pure host overhead:
Python validation + ctypes + the C ABI's plan/encode/launch), and for the
given size the per-call time of (a) single calls bracketed by events (host
overhead + kernel), (b) 50 back-to-back calls between two events, (c) the
same 50 calls replayed from a CUDA graph (kernel + launch gaps only).
"""
import argparse
import statistics
import sys
import time
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--n", type=int, default=256)
    ap.add_argument("--fmt", default="u8")
    ap.add_argument("--k", type=int, default=3)
    ap.add_argument("--mode", default="clamp")
    args = ap.parse_args()
    import torch

    import paper_2203_10213_b200 as vk

    fmt = vk.DataFormat.parse(args.fmt)
    k = vk.gaussian_kernel(1.0, args.k)

    def vols(n):
        s = vk.synthetic_device((n, n, n), fmt, seed=7)
        d = vk.StructuredVolume(s.dims, fmt, data=vk.DeviceBuffer(s.nbytes, zero=False))
        return s, d

    s16, d16 = vols(16)
    for _ in range(20):
        vk.ApplyFilter(d16, s16, k, args.mode)
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(2000):
        vk.ApplyFilter(d16, s16, k, args.mode)
    t1 = time.perf_counter()
    torch.cuda.synchronize()
    print(f"host overhead per ApplyFilter call (16^3): {(t1 - t0) / 2000 * 1e6:.1f} us")

    src, dst = vols(args.n)
    st = torch.cuda.current_stream()
    for _ in range(5):
        vk.ApplyFilter(dst, src, k, args.mode)
    single = []
    for _ in range(20):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(st)
        vk.ApplyFilter(dst, src, k, args.mode)
        b.record(st)
        b.synchronize()
        single.append(a.elapsed_time(b) * 1e3)
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record(st)
    for _ in range(50):
        vk.ApplyFilter(dst, src, k, args.mode)
    b.record(st)
    b.synchronize()
    batch = a.elapsed_time(b) * 1e3 / 50
    g = torch.cuda.CUDAGraph()
    side = torch.cuda.Stream()
    side.wait_stream(st)
    with torch.cuda.stream(side):
        with torch.cuda.graph(g, stream=side):
            for _ in range(50):
                vk.ApplyFilter(dst, src, k, args.mode)
    st.wait_stream(side)
    g.replay()
    torch.cuda.synchronize()
    a.record(st)
    g.replay()
    b.record(st)
    b.synchronize()
    graph = a.elapsed_time(b) * 1e3 / 50
    nv = args.n ** 3
    print(f"{args.fmt} k={args.k} {args.n}^3 {args.mode}: single-call events best {min(single):.1f} us "
          f"median {statistics.median(single):.1f} us; 50 back-to-back {batch:.1f} us/call "
          f"({nv / batch / 1e3:.1f} GVox/s); CUDA graph {graph:.1f} us/call ({nv / graph / 1e3:.1f} GVox/s)")


if __name__ == "__main__":
    main()
