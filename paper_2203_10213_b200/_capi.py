"""ctypes binding of the C ABI in include/vkt_b200.h (libvkt_b200.so).

This is the whole Python↔native boundary: plain pointers, sizes and a CUDA
stream handle; no torch types cross it.  The library is built in-tree by
``paper_2203_10213_b200/build.py``.  There is no CPU fallback: if the library
is missing, every device call raises ``DeviceFailure``.
"""

from __future__ import annotations

import ctypes
import os
import threading
from pathlib import Path

from .errors import DeviceFailure, from_status_name

# VKT_LIB: load a diagnostics build (build.py --variant=...) instead
LIB_PATH = Path(os.environ.get("VKT_LIB") or Path(__file__).resolve().parent / "libvkt_b200.so")

# enums (vkt_b200.h)
U8, U16, F32 = 1, 2, 3
WRAP, MIRROR, CLAMP, BORDER = 0, 1, 2, 3
FLAG_EXACT_F64 = 1
FLAG_FORCE_DIRECT = 2
FLAG_HOST_BOUNDED = 4
FLAG_NO_SEPARABLE = 8
PATH_NONE, PATH_DIRECT, PATH_EXACT, PATH_TMA, PATH_SEPARABLE = 0, 1, 2, 3, 4
PATH_NAMES = {PATH_NONE: "none", PATH_DIRECT: "direct", PATH_EXACT: "exact", PATH_TMA: "tma",
              PATH_SEPARABLE: "separable"}

EXPORTED_SYMBOLS = (
    "vkt_apply_filter",
    "vkt_apply_filter_host",
    "vkt_filter_path",
    "vkt_filter_chunk_planes",
    "vkt_fill_box",
    "vkt_fill_synthetic",
    "vkt_status_name",
    "vkt_last_error_detail",
    "vkt_launch_count",
    "vkt_abi_version",
    "vkt_clahe_histograms",
    "vkt_clahe_blend",
    "vkt_flip",
    "vkt_resample",
)


class Int3(ctypes.Structure):
    _fields_ = [("x", ctypes.c_int32), ("y", ctypes.c_int32), ("z", ctypes.c_int32)]


class FilterArgs(ctypes.Structure):
    _fields_ = [
        ("src", ctypes.c_void_p),
        ("dst", ctypes.c_void_p),
        ("dims", Int3),
        ("format", ctypes.c_int32),
        ("map_lo", ctypes.c_double),
        ("map_hi", ctypes.c_double),
        ("weights", ctypes.POINTER(ctypes.c_double)),
        ("kdims", Int3),
        ("address_mode", ctypes.c_int32),
        ("halo_lo", ctypes.c_void_p),
        ("halo_hi", ctypes.c_void_p),
        ("z_offset", ctypes.c_int64),
        ("global_nz", ctypes.c_int64),
        ("out_z_begin", ctypes.c_int32),
        ("out_z_end", ctypes.c_int32),
        ("flags", ctypes.c_int32),
    ]


_lib = None
_lock = threading.Lock()


def load(path: Path | str | None = None) -> ctypes.CDLL:
    """Load (once) and type the shared library; raises DeviceFailure if absent."""
    global _lib
    with _lock:
        if _lib is not None and path is None:
            return _lib
        p = Path(path) if path is not None else LIB_PATH
        if not p.exists():
            raise DeviceFailure(
                f"{p} is not built; run `python -c 'import __graft_entry__ as g; g.build()'` "
                "(there is no CPU fallback)"
            )
        lib = ctypes.CDLL(str(p))
        vp, i32, i64, u32, u64 = (ctypes.c_void_p, ctypes.c_int32, ctypes.c_int64,
                                  ctypes.c_uint32, ctypes.c_uint64)
        lib.vkt_apply_filter.argtypes = [ctypes.POINTER(FilterArgs), vp]
        lib.vkt_apply_filter.restype = ctypes.c_int
        lib.vkt_apply_filter_host.argtypes = [ctypes.POINTER(FilterArgs), ctypes.c_int32, vp]
        lib.vkt_apply_filter_host.restype = ctypes.c_int
        lib.vkt_filter_path.argtypes = [ctypes.POINTER(FilterArgs)]
        lib.vkt_filter_path.restype = ctypes.c_int
        lib.vkt_filter_chunk_planes.argtypes = [ctypes.POINTER(FilterArgs)]
        lib.vkt_filter_chunk_planes.restype = ctypes.c_int
        lib.vkt_fill_box.argtypes = [vp, Int3, i32, Int3, Int3, u32, vp]
        lib.vkt_fill_box.restype = ctypes.c_int
        lib.vkt_fill_synthetic.argtypes = [vp, Int3, i32, u64, i64, vp]
        lib.vkt_fill_synthetic.restype = ctypes.c_int
        lib.vkt_status_name.argtypes = [ctypes.c_int]
        lib.vkt_status_name.restype = ctypes.c_char_p
        lib.vkt_last_error_detail.argtypes = []
        lib.vkt_last_error_detail.restype = ctypes.c_char_p
        lib.vkt_launch_count.argtypes = []
        lib.vkt_launch_count.restype = u64
        lib.vkt_abi_version.argtypes = []
        lib.vkt_abi_version.restype = ctypes.c_int
        if path is None:
            _lib = lib
        return lib


def check(status: int) -> None:
    """Raise the reference-named VktError for a non-zero status."""
    if status == 0:
        return
    lib = load()
    name = lib.vkt_status_name(status).decode()
    detail = lib.vkt_last_error_detail().decode()
    raise from_status_name(name, detail)


def launch_count() -> int:
    return int(load().vkt_launch_count())


def int3(v) -> Int3:
    x, y, z = v
    return Int3(int(x), int(y), int(z))
