"""ApplyFilter: 3D correlation of a StructuredVolume on the B200.

Reference: ``apply_filter(volume, kernel)`` (pkg/src/vkt/ops/filters.py:69-95)
correlates (no kernel flip) in mapped-value space against an immutable
snapshot with clamp-to-edge reads and re-quantizes in place.  This module
keeps that call and its ``Kernel`` / ``gaussian_kernel`` / ``box_kernel``
helpers (filters.py:23-66) and adds the north star's
``ApplyFilter(dst, src, filter, address_mode)`` with the Wrap / Mirror /
Clamp / Border modes.  All arithmetic happens in ``libvkt_b200.so``
(include/vkt_b200.h); this file only validates, packs arguments and picks
the stream.  There is no CPU fallback.
"""

from __future__ import annotations

import ctypes
import math
from enum import IntEnum

import numpy as np

from . import _capi
from .errors import EvenKernelDims, InvalidArgument
from .execution import FilterPath, debug, get_execution_policy, timed
from .geom import Vec3i, ivec3
from .volume import DataFormat, StructuredVolume, require_same_layout


class AddressMode(IntEnum):
    """Boundary handling; values match VKT_WRAP.. in include/vkt_b200.h."""

    WRAP = 0     # i mod n                      (np.pad "wrap")
    MIRROR = 1   # edge-duplicating reflection  (np.pad "symmetric")
    CLAMP = 2    # clamp-to-edge: the reference (np.pad "edge", filters.py:78)
    BORDER = 3   # stored value 0               (np.pad "constant")

    @classmethod
    def coerce(cls, v) -> "AddressMode":
        if isinstance(v, AddressMode):
            return v
        if isinstance(v, str):
            try:
                return cls[v.strip().upper()]
            except KeyError:
                raise InvalidArgument(f"unknown address mode {v!r}") from None
        try:
            return cls(int(v))
        except ValueError:
            raise InvalidArgument(f"unknown address mode {v!r}") from None


class Kernel:
    """Dense correlation kernel with odd extent per axis (filters.py:23-43).

    ``weights`` is float64 shaped (kz, ky, kx), built from an x-fastest flat
    sequence exactly like the reference's reshape (filters.py:34-36).
    """

    def __init__(self, dims, weights):
        self.dims = ivec3(dims, "kernel dims")
        if any(d < 1 or d % 2 == 0 for d in self.dims):
            raise EvenKernelDims(f"kernel dims must be odd, got {tuple(self.dims)}")
        try:
            w = np.asarray(weights, dtype=np.float64).reshape(self.dims.z, self.dims.y, self.dims.x)
        except ValueError as e:
            raise InvalidArgument(f"kernel weights do not match dims {tuple(self.dims)}: {e}") from None
        if not np.isfinite(w).all():
            raise InvalidArgument("kernel weights must be finite")
        self.weights = w

    @property
    def radius(self) -> Vec3i:
        d = self.dims
        return Vec3i(d.x // 2, d.y // 2, d.z // 2)

    @property
    def tap_count(self) -> int:
        d = self.dims
        return d.x * d.y * d.z

    def __repr__(self):
        return f"Kernel(dims={tuple(self.dims)})"


#: The north star calls the kernel a Filter; same type.
Filter = Kernel


def gaussian_kernel(sigma: float, size: int | None = None) -> Kernel:
    """Normalized isotropic Gaussian (filters.py:46-59).

    Same float64 operation sequence as the reference so the weights are
    bit-identical: separable exp profile, outer product (z, y, x), divided by
    the numpy sum.  Default extent 2*ceil(2*sigma)+1.
    """
    if not sigma > 0:
        raise InvalidArgument(f"sigma must be > 0, got {sigma}")
    if size is None:
        size = 2 * int(math.ceil(2.0 * sigma)) + 1
    if size % 2 == 0:
        raise EvenKernelDims(f"kernel size must be odd, got {size}")
    r = size // 2
    t = np.arange(-r, r + 1, dtype=np.float64)
    prof = np.exp(-0.5 * (t / sigma) ** 2)
    w = prof[:, None, None] * prof[None, :, None] * prof[None, None, :]
    w /= w.sum()
    return Kernel((size, size, size), w)


def box_kernel(size: int) -> Kernel:
    """Uniform kernel 1/size^3 (filters.py:62-66)."""
    if size % 2 == 0:
        raise EvenKernelDims(f"kernel size must be odd, got {size}")
    return Kernel((size, size, size), np.full((size, size, size), 1.0 / size**3))


def laplacian_kernel() -> Kernel:
    """7-point Laplacian in a dense 3^3 footprint (centre -6, faces +1).

    Not in the reference; BASELINE config 4 uses it.  All 27 taps are
    evaluated, like the reference would.
    """
    w = np.zeros((3, 3, 3))
    w[1, 1, 1] = -6.0
    for z, y, x in ((0, 1, 1), (2, 1, 1), (1, 0, 1), (1, 2, 1), (1, 1, 0), (1, 1, 2)):
        w[z, y, x] = 1.0
    return Kernel((3, 3, 3), w)


def _flags(policy) -> int:
    if policy.filter_path is FilterPath.EXACT:
        return _capi.FLAG_EXACT_F64
    if policy.filter_path is FilterPath.DIRECT:
        return _capi.FLAG_FORCE_DIRECT
    if policy.filter_path is FilterPath.DENSE:
        return _capi.FLAG_NO_SEPARABLE
    return 0


def make_args(dst_ptr: int, src_ptr: int, dims, fmt: DataFormat, mapping, kernel: Kernel,
              mode: AddressMode, *, halo_lo: int = 0, halo_hi: int = 0, z_offset: int = 0,
              global_nz: int = 0, out_z_begin: int = 0, out_z_end: int = 0,
              flags: int = 0):
    """Pack a ``vkt_filter_args``; returns (args, keepalive) — keep both alive."""
    # The flat float64 weights, their pointer and the kernel extents are cached
    # on the kernel (keyed on the weights array object; the flat array is a
    # view, so in-place edits of kernel.weights are seen): repacking them cost
    # a third of the per-call host time.
    cached = kernel.__dict__.get("_abi")
    if cached is None or cached[0] is not kernel.weights:
        flat = np.ascontiguousarray(kernel.weights.reshape(-1), dtype=np.float64)
        cached = (kernel.weights, flat, flat.ctypes.data_as(ctypes.POINTER(ctypes.c_double)),
                  _capi.int3(kernel.dims))
        kernel.__dict__["_abi"] = cached
    _, w, wptr, kd = cached
    lo, hi = mapping
    x, y, z = dims
    # one positional constructor call (field order of vkt_filter_args)
    a = _capi.FilterArgs(src_ptr, dst_ptr, _capi.Int3(int(x), int(y), int(z)), fmt.value, float(lo),
                         float(hi), wptr, kd, int(mode), halo_lo or None, halo_hi or None,
                         int(z_offset), int(global_nz), int(out_z_begin), int(out_z_end), int(flags))
    return a, w


def launch(args, stream_handle: int) -> None:
    """Call ``vkt_apply_filter`` and raise the reference-named error on failure."""
    lib = _capi.load()
    _capi.check(lib.vkt_apply_filter(ctypes.byref(args), ctypes.c_void_p(stream_handle)))


def filter_path(dst: StructuredVolume, src: StructuredVolume, kernel: Kernel,
                address_mode=AddressMode.CLAMP) -> str:
    """Which kernel ApplyFilter would launch ("separable", "tma", "direct",
    "exact")."""
    mode = AddressMode.coerce(address_mode)
    args, _keep = make_args(dst.data_ptr(), src.data_ptr(), src.dims, src.format, src.mapping,
                            kernel, mode, flags=_flags(get_execution_policy()))
    return _capi.PATH_NAMES[_capi.load().vkt_filter_path(ctypes.byref(args))]


def chunk_planes(src: StructuredVolume, kernel: Kernel, address_mode=AddressMode.CLAMP) -> int:
    """Output planes per CTA z-chunk the tiled kernel uses for this launch
    (0 when another kernel runs).  Chunk boundaries restart a CTA's rolling z
    accumulators; the at-size parity tests probe both sides of each."""
    import torch

    mode = AddressMode.coerce(address_mode)
    args, _keep = make_args(src.data_ptr(), src.data_ptr() + 16, src.dims, src.format, src.mapping,
                            kernel, mode, flags=_flags(get_execution_policy()))
    with torch.cuda.device(src.data.device):
        return int(_capi.load().vkt_filter_chunk_planes(ctypes.byref(args)))


def _current_stream(volume: StructuredVolume) -> int:
    import torch

    return int(torch.cuda.current_stream(volume.data.device).cuda_stream)


@timed("ApplyFilter")
def ApplyFilter(dst: StructuredVolume, src: StructuredVolume, filter: Kernel,
                address_mode=AddressMode.CLAMP) -> None:
    """dst = correlate(src, filter) under ``address_mode``, re-quantized to dst's format.

    ``dst`` and ``src`` must agree in dims, format and mapping.  Passing the
    same volume twice filters in place (snapshot semantics, filters.py:77).
    Volumes in HBM: asynchronous on the current torch CUDA stream.
    Host-resident volumes (``Device.CPU``): streamed through HBM by the
    host-buffer pipeline; returns when ``dst`` holds the result.
    """
    if not isinstance(filter, Kernel):
        raise InvalidArgument("filter must be a Kernel/Filter")
    mode = AddressMode.coerce(address_mode)
    if dst is src:
        _apply_in_place(src, filter, mode)
        return
    src.data.migrate()
    dst.data.migrate()
    require_same_layout(dst, src)
    policy = get_execution_policy()
    if policy.debug_messages:
        debug(f"ApplyFilter {src!r} k={tuple(filter.dims)} mode={mode.name}")
    if src.on_host:
        _apply_host_resident(dst, src, filter, mode)
        return
    args, _keep = make_args(dst.data_ptr(), src.data_ptr(), src.dims, src.format, src.mapping,
                            filter, mode, flags=_flags(policy))
    launch(args, _current_stream(src))


def _apply_host_resident(dst: StructuredVolume, src: StructuredVolume, kernel: Kernel,
                         mode: AddressMode) -> None:
    """Both volumes in page-locked host memory: the chunked H2D / filter / D2H
    pipeline of ``vkt_apply_filter_host`` (csrc/vkt_host.cu) on the device."""
    d = src.dims
    shape = (d.z, d.y, d.x)
    s_arr = src.data.array.view(src.format.dtype).reshape(shape)
    d_arr = dst.data.array.view(dst.format.dtype).reshape(shape)
    apply_filter_host(s_arr, kernel, mode, fmt=src.format, mapping=tuple(src.mapping), out=d_arr)


def _apply_in_place(volume: StructuredVolume, kernel: Kernel, mode: AddressMode) -> None:
    import torch

    volume.data.migrate()
    out = StructuredVolume(volume.dims, volume.format, volume.cell_size, volume.mapping,
                           data=volume.data.empty_like())
    if volume.on_host:
        _apply_host_resident(out, volume, kernel, mode)
        volume.swap_storage(out)
        return
    args, _keep = make_args(out.data_ptr(), volume.data_ptr(), volume.dims, volume.format,
                            volume.mapping, kernel, mode, flags=_flags(get_execution_policy()))
    stream = torch.cuda.current_stream(volume.data.device)
    launch(args, int(stream.cuda_stream))
    # The old bytes go back to the torch caching allocator; recording the
    # launch stream keeps them from being reused before the kernel has read them.
    volume.data.tensor.record_stream(stream)
    volume.swap_storage(out)


@timed("ApplyFilter")
def apply_filter(volume: StructuredVolume, kernel: Kernel, address_mode=AddressMode.CLAMP) -> None:
    """In-place filter with the reference's signature (filters.py:69-95).

    The reference always clamps; ``address_mode`` is an optional extension.
    """
    if not isinstance(kernel, Kernel):
        raise InvalidArgument("kernel must be a Kernel")
    _apply_in_place(volume, kernel, AddressMode.coerce(address_mode))


def apply_filter_host(stored, kernel: Kernel, address_mode=AddressMode.CLAMP, *, fmt=None,
                      mapping=(0.0, 1.0), out=None, z_range=None, chunk_planes: int = 0,
                      z_offset: int = 0, global_nz: int = 0, halo_lo=None, halo_hi=None,
                      bounded_memory: bool = False):
    """ApplyFilter on a HOST (z, y, x) array, streamed through HBM.

    The reference filters host numpy arrays (filters.py:69-95); this keeps that
    contract without a device-resident volume: ``vkt_apply_filter_host``
    uploads z-chunks plus their halo planes, filters and downloads them with
    the three phases overlapped (page-locked arrays, e.g. numpy views of
    ``torch.empty(..., pin_memory=True)``, make the copies asynchronous).
    Returns ``out`` (a new array of the input dtype unless given); only the
    output planes ``z_range`` (default all) are written.  Bit-identical to
    ``ApplyFilter`` on the whole volume; volumes larger than HBM work.

    ``z_offset`` / ``global_nz``: the array holds global planes
    [z_offset, z_offset + nz) of a volume with ``global_nz`` planes (a z-slab
    read with range I/O, or one rank's share); every halo plane the requested
    outputs need must be inside it, unless ``halo_lo`` / ``halo_hi`` (host
    arrays of rz = kz//2 planes: the address-mapped planes just below and
    above the array) supply them.  ``z_range`` is relative to the array.

    The padded input is kept resident on the device when it fits in half the
    free HBM (each chunk uploads only its new planes); ``bounded_memory``
    streams it through a few chunk-sized ring buffers instead.
    """
    import torch

    if not isinstance(kernel, Kernel):
        raise InvalidArgument("kernel must be a Kernel")
    src = np.asarray(stored)
    if src.ndim != 3 or not src.flags["C_CONTIGUOUS"]:
        raise InvalidArgument("apply_filter_host needs a C-contiguous (z, y, x) array")
    if fmt is None:
        fmt = {np.dtype("<u1"): DataFormat.UINT8, np.dtype("<u2"): DataFormat.UINT16,
               np.dtype("<f4"): DataFormat.FLOAT32}.get(src.dtype.newbyteorder("<") if src.dtype.byteorder == ">" else src.dtype)
        if fmt is None:
            raise InvalidArgument(f"no voxel format for dtype {src.dtype}")
    fmt = fmt if isinstance(fmt, DataFormat) else DataFormat.parse(fmt)
    if src.dtype != fmt.dtype:
        raise InvalidArgument(f"array dtype {src.dtype} does not match format {fmt.short_name}")
    if out is None:
        out = np.empty_like(src)
    elif out.shape != src.shape or out.dtype != src.dtype or not out.flags["C_CONTIGUOUS"]:
        raise InvalidArgument("out must match the input's shape and dtype and be C-contiguous")
    nz, ny, nx = src.shape
    zb, ze = (0, 0) if z_range is None else (int(z_range[0]), int(z_range[1]))
    mode = AddressMode.coerce(address_mode)
    halos = []
    for h in (halo_lo, halo_hi):
        if h is None:
            halos.append(0)
            continue
        h = np.asarray(h)
        if (h.dtype != src.dtype or not h.flags["C_CONTIGUOUS"]
                or h.shape != (kernel.radius.z, ny, nx)):
            raise InvalidArgument(f"halo arrays must be C-contiguous ({kernel.radius.z}, {ny}, {nx}) "
                                  f"{src.dtype}")
        halos.append(h.ctypes.data)
    args, _keep = make_args(out.ctypes.data, src.ctypes.data, (nx, ny, nz), fmt, mapping, kernel, mode,
                            out_z_begin=zb, out_z_end=ze, z_offset=z_offset, global_nz=global_nz,
                            halo_lo=halos[0], halo_hi=halos[1],
                            flags=_flags(get_execution_policy()) | (_capi.FLAG_HOST_BOUNDED if bounded_memory else 0))
    stream = int(torch.cuda.current_stream().cuda_stream) if torch.cuda.is_available() else 0
    _capi.check(_capi.load().vkt_apply_filter_host(ctypes.byref(args), int(chunk_planes),
                                                   ctypes.c_void_p(stream)))
    return out
