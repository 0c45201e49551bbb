"""Compute-side cost of the sharded schedule on ONE GPU (no communication):
one rank's slab of a P-way z split, with halo buffers, filtered
(a) as one launch over all output planes, and
(b) as the sharded schedule does it: interior launch + two boundary launches.

  python tools/shard_overhead.py [--p 8] [--fmt u16] [--k 7] [--n 1024]
"""
import argparse
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--p", type=int, default=8)
    ap.add_argument("--fmt", default="u16")
    ap.add_argument("--k", type=int, default=7)
    ap.add_argument("--n", type=int, default=1024)
    ap.add_argument("--reps", type=int, default=10)
    args = ap.parse_args()
    import torch

    import paper_2203_10213_b200 as vk
    from paper_2203_10213_b200.filters import launch, make_args

    fmt = vk.DataFormat.parse(args.fmt)
    k = vk.gaussian_kernel(1.5 if args.k == 7 else 1.0, args.k)
    n = args.n
    nz = n // args.p
    rz = args.k // 2
    src = vk.synthetic_device((n, n, nz), fmt, seed=7)
    dst = vk.StructuredVolume(src.dims, fmt, data=vk.DeviceBuffer(src.nbytes, zero=False))
    lo = vk.synthetic_device((n, n, rz), fmt, seed=8)
    hi = vk.synthetic_device((n, n, rz), fmt, seed=9)
    st = torch.cuda.current_stream()
    common = dict(dims=(n, n, nz), fmt=fmt, mapping=(0.0, 1.0), kernel=k, mode=vk.AddressMode.CLAMP,
                  z_offset=nz * (args.p // 2), global_nz=n, halo_lo=lo.data_ptr(), halo_hi=hi.data_ptr())

    def run(ranges):
        for b, e in ranges:
            a, _w = make_args(dst.data_ptr(), src.data_ptr(), **common, out_z_begin=b, out_z_end=e)
            launch(a, int(st.cuda_stream))

    def timeit(ranges):
        for _ in range(3):
            run(ranges)
        best = 1e9
        for _ in range(args.reps):
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(st)
            run(ranges)
            e1.record(st)
            e1.synchronize()
            best = min(best, e0.elapsed_time(e1))
        return best

    side = torch.cuda.Stream()

    def run_concurrent():
        side.wait_stream(st)
        a, _w = make_args(dst.data_ptr(), src.data_ptr(), **common, out_z_begin=rz, out_z_end=nz - rz)
        launch(a, int(st.cuda_stream))
        for b, e in ((0, rz), (nz - rz, nz)):
            a, _w = make_args(dst.data_ptr(), src.data_ptr(), **common, out_z_begin=b, out_z_end=e)
            launch(a, int(side.cuda_stream))
        st.wait_stream(side)

    for _ in range(3):
        run_concurrent()
    conc = 1e9
    for _ in range(args.reps):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(st)
        run_concurrent()
        e1.record(st)
        e1.synchronize()
        conc = min(conc, e0.elapsed_time(e1))
    full = timeit([(0, nz)])
    split = timeit([(rz, nz - rz), (0, rz), (nz - rz, nz)])
    inner = timeit([(rz, nz - rz)])
    bnd = timeit([(0, rz), (nz - rz, nz)])
    print(f"P={args.p} slab {n}x{n}x{nz} {args.fmt} k={args.k}: one launch {full:.3f} ms; "
          f"interior+2 boundary {split:.3f} ms (interior {inner:.3f}, boundaries {bnd:.3f}); "
          f"overhead {100 * (split / full - 1):.1f}%; boundaries on a second stream beside the interior "
          f"{conc:.3f} ms (overhead {100 * (conc / full - 1):.1f}%)")


if __name__ == "__main__":
    main()
