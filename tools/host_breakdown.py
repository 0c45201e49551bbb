"""Where the ~15 us of host time per ApplyFilter call goes (16^3 u8, 3^3)."""
import ctypes
import sys
import time
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))


def per_call(fn, n=4000):
    for _ in range(200):
        fn()
    t0 = time.perf_counter()
    for _ in range(n):
        fn()
    return (time.perf_counter() - t0) / n * 1e6


def main():
    import torch

    import paper_2203_10213_b200 as vk
    from paper_2203_10213_b200 import _capi
    from paper_2203_10213_b200.filters import _current_stream, make_args

    src = vk.synthetic_device((16, 16, 16), vk.DataFormat.UINT8, seed=7)
    dst = vk.StructuredVolume(src.dims, src.format)
    k = vk.gaussian_kernel(1.0, 3)
    lib = _capi.load()
    a, keep = make_args(dst.data_ptr(), src.data_ptr(), src.dims, src.format, src.mapping, k,
                        vk.AddressMode.CLAMP)
    sh = _current_stream(src)
    rows = {
        "ApplyFilter (public API)": lambda: vk.ApplyFilter(dst, src, k, vk.AddressMode.CLAMP),
        "make_args": lambda: make_args(dst.data_ptr(), src.data_ptr(), src.dims, src.format, src.mapping,
                                       k, vk.AddressMode.CLAMP),
        "_current_stream": lambda: _current_stream(src),
        "data_ptr x2": lambda: (dst.data_ptr(), src.data_ptr()),
        "vkt_filter_path (C plan, no launch)": lambda: lib.vkt_filter_path(ctypes.byref(a)),
        "vkt_apply_filter (C plan + encode + launch)": lambda: lib.vkt_apply_filter(ctypes.byref(a), ctypes.c_void_p(sh)),
    }
    for name, fn in rows.items():
        print(f"{per_call(fn):7.2f} us  {name}")
    vk.set_execution_policy(vk.ExecutionPolicy(filter_path="dense"))
    a2, keep2 = make_args(dst.data_ptr(), src.data_ptr(), src.dims, src.format, src.mapping, k,
                          vk.AddressMode.CLAMP, flags=_capi.FLAG_NO_SEPARABLE)
    print(f"{per_call(lambda: lib.vkt_apply_filter(ctypes.byref(a2), ctypes.c_void_p(sh))):7.2f} us  "
          "vkt_apply_filter, dense path")
    print(f"{per_call(lambda: vk.ApplyFilter(dst, src, k, vk.AddressMode.CLAMP)):7.2f} us  ApplyFilter, dense path")
    vk.set_execution_policy(vk.ExecutionPolicy())
    torch.cuda.synchronize()


if __name__ == "__main__":
    main()
