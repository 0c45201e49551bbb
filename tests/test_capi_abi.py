"""CPU: the C-ABI library loads and exports every symbol include/vkt_b200.h declares.

Only calls that return before touching the device are made here (argument
validation); kernels need a GPU and live in the gpu-marked tests.
"""

import ctypes
import re
from pathlib import Path

import numpy as np
import pytest

from paper_2203_10213_b200 import _capi

HEADER = Path(__file__).resolve().parent.parent / "include" / "vkt_b200.h"


def declared_functions():
    text = HEADER.read_text()
    text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
    return sorted(set(re.findall(r"\b(vkt_[a-z_0-9]+)\s*\(", text)))


@pytest.fixture(scope="module")
def lib():
    if not _capi.LIB_PATH.exists():
        from paper_2203_10213_b200 import build

        build.build()
    return _capi.load()


def test_exports_every_declared_symbol(lib):
    decl = declared_functions()
    assert set(decl) == set(_capi.EXPORTED_SYMBOLS)
    for name in decl:
        assert hasattr(lib, name), name


def test_status_names_follow_reference_errors(lib):
    assert lib.vkt_status_name(0) == b"OK"
    assert lib.vkt_status_name(1) == b"InvalidArgument"
    assert lib.vkt_status_name(2) == b"EvenKernelDims"
    assert lib.vkt_status_name(3) == b"AllocationFailure"
    assert lib.vkt_status_name(4) == b"DeviceFailure"
    assert lib.vkt_abi_version() >= 10000


def _args(**over):
    w = np.full(27, 1 / 27.0)
    a = _capi.FilterArgs()
    a.src, a.dst = 0x1000, 0x2000  # never dereferenced: validation fails first
    a.dims = _capi.Int3(8, 8, 8)
    a.format = 1
    a.map_lo, a.map_hi = 0.0, 1.0
    a.weights = w.ctypes.data_as(ctypes.POINTER(ctypes.c_double))
    a.kdims = _capi.Int3(3, 3, 3)
    a.address_mode = 2
    for k, v in over.items():
        setattr(a, k, v)
    return a, w


@pytest.mark.parametrize("over,status", [
    (dict(kdims=_capi.Int3(2, 3, 3)), 2),
    (dict(kdims=_capi.Int3(3, 3, 0)), 2),
    (dict(dims=_capi.Int3(0, 8, 8)), 1),
    (dict(format=7), 1),
    (dict(address_mode=9), 1),
    (dict(map_lo=1.0, map_hi=1.0), 1),
    (dict(dst=0x1000), 1),            # aliasing src
    (dict(global_nz=64, z_offset=8), 1),  # sharded slab without halos
    (dict(global_nz=12, z_offset=8), 1),  # slab outside global extent
])
def test_validation_errors(lib, over, status):
    a, _w = _args(**over)
    assert lib.vkt_apply_filter(ctypes.byref(a), None) == status
    assert lib.vkt_filter_path(ctypes.byref(a)) == 0
    with pytest.raises(Exception) as ei:
        _capi.check(status)
    assert type(ei.value).__name__ == lib.vkt_status_name(status).decode()


def test_nonfinite_weight_rejected(lib):
    a, w = _args()
    w[5] = np.inf
    assert lib.vkt_apply_filter(ctypes.byref(a), None) == 1
    assert b"finite" in lib.vkt_last_error_detail()


def test_path_selection_is_host_logic(lib):
    a, _w = _args()
    assert lib.vkt_filter_path(ctypes.byref(a)) in (_capi.PATH_DIRECT, _capi.PATH_TMA)
    a.flags = _capi.FLAG_EXACT_F64
    assert lib.vkt_filter_path(ctypes.byref(a)) == _capi.PATH_EXACT
    a.flags = _capi.FLAG_FORCE_DIRECT
    assert lib.vkt_filter_path(ctypes.byref(a)) == _capi.PATH_DIRECT


def test_fill_box_validation(lib):
    assert lib.vkt_fill_box(None, _capi.Int3(4, 4, 4), 1, _capi.Int3(0, 0, 0),
                            _capi.Int3(4, 4, 4), 0, None) == 1
    assert lib.vkt_fill_box(0x1000, _capi.Int3(4, 4, 4), 5, _capi.Int3(0, 0, 0),
                            _capi.Int3(4, 4, 4), 0, None) == 1
    # empty roi is a no-op that succeeds without touching the device (core.py:48-49)
    assert lib.vkt_fill_box(0x1000, _capi.Int3(4, 4, 4), 1, _capi.Int3(2, 2, 2),
                            _capi.Int3(2, 2, 2), 0, None) == 0
