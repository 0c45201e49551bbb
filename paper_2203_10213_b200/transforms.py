"""Flip and Resample of structured volumes on the B200.

The remaining structured-volume members of the paper's §4.3 benchmark
assortment next to ApplyFilter (the reference bench cases
``resample_down2`` and ``flip_longest_axis``, bench.py:110-117).

* ``flip(volume, axis)``  — pkg/src/vkt/ops/geometric.py:34-40: reverse the
  stored cells along x / y / z; a permutation, bit-exact.
* ``resample(source, dst_dims, dst_format=None, dst_mapping=None)`` —
  pkg/src/vkt/ops/core.py:202-262: trilinear samples of the mapped grid at the
  destination cell centers (clamp-to-edge, volume.py:237-266), re-quantized;
  float64 in numpy's operation order, bit-identical to the reference.
"""

from __future__ import annotations

import ctypes

import numpy as np

from . import _capi
from .errors import InvalidArgument
from .execution import timed
from .geom import Vec3i
from .volume import DataFormat, DeviceBuffer, StructuredVolume, VoxelMapping, device_resident

_AXES = {"x": 0, "y": 1, "z": 2}


def _axis(axis) -> int:
    if isinstance(axis, str):
        key = axis.strip().lower()
        if key not in _AXES:
            raise InvalidArgument(f"unknown axis {axis!r}")
        return _AXES[key]
    if axis not in (0, 1, 2):
        raise InvalidArgument(f"axis must be x, y, z or 0, 1, 2, got {axis!r}")
    return int(axis)


def _lib():
    lib = _capi.load()
    if not getattr(lib, "_xform_typed", False):
        vp, i32, d = ctypes.c_void_p, ctypes.c_int32, ctypes.c_double
        lib.vkt_flip.argtypes = [vp, vp, _capi.Int3, i32, i32, vp]
        lib.vkt_flip.restype = ctypes.c_int
        lib.vkt_resample.argtypes = [vp, _capi.Int3, i32, d, d, vp, _capi.Int3, i32, d, d, vp]
        lib.vkt_resample.restype = ctypes.c_int
        lib._xform_typed = True
    return lib


def _stream(volume):
    import torch

    return ctypes.c_void_p(int(torch.cuda.current_stream(volume.data.device).cuda_stream))


@timed("Flip")
def flip(volume: StructuredVolume, axis) -> None:
    """Reverse stored values along one axis, in place (geometric.py:34-40)."""
    import torch

    a = _axis(axis)
    with device_resident(volume) as v:
        out = StructuredVolume(v.dims, v.format, v.cell_size, v.mapping, data=v.data.empty_like())
        _capi.check(_lib().vkt_flip(v.data_ptr(), out.data_ptr(), _capi.int3(v.dims),
                                    v.format.value, a, _stream(v)))
        v.data.tensor.record_stream(torch.cuda.current_stream(v.data.device))
        v.swap_storage(out)


@timed("Resample")
def resample(source: StructuredVolume, dst_dims, dst_format=None, dst_mapping=None) -> StructuredVolume:
    """Resample onto a grid of `dst_dims` cells keeping the world extent (core.py:202-262)."""
    if not isinstance(source, StructuredVolume):
        raise InvalidArgument("resample takes a structured volume (hierarchical volumes are out of scope)")
    dst_dims = Vec3i(*(int(v) for v in dst_dims))
    if min(dst_dims) < 1:
        raise InvalidArgument(f"resample target dims must be >= 1, got {tuple(dst_dims)}")
    fmt = source.format if dst_format is None else (
        dst_format if isinstance(dst_format, DataFormat) else DataFormat.parse(dst_format))
    mapping = source.mapping if dst_mapping is None else VoxelMapping.coerce(dst_mapping)
    src_cell = np.asarray(source.cell_size, dtype=np.float64)
    dst_cell = src_cell * np.asarray(source.dims, dtype=np.float64) / np.asarray(dst_dims, dtype=np.float64)
    nbytes = dst_dims.x * dst_dims.y * dst_dims.z * fmt.bytes_per_cell
    with device_resident(source, write_back=False) as src:
        out = StructuredVolume(dst_dims, fmt, tuple(dst_cell), mapping,
                               data=DeviceBuffer(nbytes, device=src.data.device, zero=False))
        _capi.check(_lib().vkt_resample(
            src.data_ptr(), _capi.int3(src.dims), src.format.value, src.mapping.lo,
            src.mapping.hi, out.data_ptr(), _capi.int3(dst_dims), fmt.value, mapping.lo, mapping.hi,
            _stream(src)))
    if source.on_host or type(source) is not StructuredVolume:
        # the result lives where the caller's volumes live (its policy's space)
        res = type(source)(dst_dims, fmt, tuple(dst_cell), mapping)
        res.data.migrate()
        res.data.raw.copy_(out.data.raw)
        return res
    return out
