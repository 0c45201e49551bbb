"""Run one ApplyFilter configuration a few times (for ncu captures).

  python tools/profile_case.py --fmt u16 --k 7 --n 1024 --mode clamp --reps 3
"""

import argparse
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--fmt", default="u16")
    ap.add_argument("--k", type=int, default=7)
    ap.add_argument("--n", type=int, default=1024)
    ap.add_argument("--nz", type=int, default=0, help="z extent (default n)")
    ap.add_argument("--mode", default="clamp")
    ap.add_argument("--kernel", default="gauss", choices=["gauss", "box", "lap"])
    ap.add_argument("--reps", type=int, default=3)
    ap.add_argument("--path", default="auto")
    args = ap.parse_args()

    import torch

    import paper_2203_10213_b200 as vk

    fmt = vk.DataFormat.parse(args.fmt)
    k = {"gauss": lambda: vk.gaussian_kernel(1.0 if args.k < 7 else 1.5, args.k),
         "box": lambda: vk.box_kernel(args.k), "lap": vk.laplacian_kernel}[args.kernel]()
    dims = (args.n, args.n, args.nz or args.n)
    src = vk.synthetic_device(dims, fmt, seed=7)
    dst = vk.StructuredVolume(src.dims, fmt, data=vk.DeviceBuffer(src.nbytes, zero=False))
    vk.set_execution_policy(vk.ExecutionPolicy(filter_path=args.path))
    s = torch.cuda.current_stream()
    times = []
    for _ in range(args.reps):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(s)
        vk.ApplyFilter(dst, src, k, args.mode)
        e1.record(s)
        e1.synchronize()
        times.append(e0.elapsed_time(e1))
    nvox = dims[0] * dims[1] * dims[2]
    best = min(times)
    print(f"{args.fmt} k={args.k} {args.kernel} dims={dims} {args.mode} path={vk.filter_path(dst, src, k, args.mode)}: "
          f"best {best:.3f} ms = {nvox / best / 1e6:.1f} GVox/s  (all: {[round(t, 3) for t in times]})")


if __name__ == "__main__":
    main()
