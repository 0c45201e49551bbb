"""Structured volumes resident in B200 HBM.

Data model of the reference (pkg/src/vkt/volume.py:29-234): a dense cell grid,
x-fastest (linear index ``i + nx*(j + ny*k)``, volume.py:3-5), little-endian
u8/u16/f32 storage, a ``VoxelMapping`` [lo, hi] for the integer formats and a
cell size.  The difference is residency: the bytes live in one CUDA
allocation (a torch ``uint8`` tensor, used purely as an allocator) instead of
a numpy arena that ``ManagedBuffer.migrate`` copies around (managed.py:97-154).
``array()`` therefore returns a *device* view shaped (z, y, x); use
``to_numpy()`` / ``from_numpy()`` at the host boundary.
"""

from __future__ import annotations

import math
from enum import Enum
from typing import Optional

import struct

import numpy as np

from .errors import AllocationFailure, DeviceFailure, IndexOutOfRange, InvalidArgument
from .execution import get_execution_policy
from .geom import Box3i, Vec3f, full_box, fvec3, ivec3


class DataFormat(Enum):
    """Voxel formats; values are the reference's format codes (volume.py:29-32)."""

    UINT8 = 1
    UINT16 = 2
    FLOAT32 = 3

    @property
    def bytes_per_cell(self) -> int:
        return _BPC[self]

    @property
    def dtype(self) -> np.dtype:
        return _NP_DTYPE[self]

    @property
    def torch_dtype(self):
        import torch

        return {DataFormat.UINT8: torch.uint8, DataFormat.UINT16: torch.uint16,
                DataFormat.FLOAT32: torch.float32}[self]

    @property
    def max_int(self) -> Optional[int]:
        return _MAX_INT[self]

    @property
    def short_name(self) -> str:
        return _SHORT[self]

    @classmethod
    def from_code(cls, code: int) -> "DataFormat":
        try:
            return cls(int(code))
        except ValueError:
            raise InvalidArgument(f"unknown data format code {code}") from None

    @classmethod
    def parse(cls, name: str) -> "DataFormat":
        key = str(name).strip().lower()
        for fmt, short in _SHORT.items():
            if key in (short, fmt.name.lower()):
                return fmt
        raise InvalidArgument(f"unknown data format {name!r}")


_BPC = {DataFormat.UINT8: 1, DataFormat.UINT16: 2, DataFormat.FLOAT32: 4}
_NP_DTYPE = {DataFormat.UINT8: np.dtype("<u1"), DataFormat.UINT16: np.dtype("<u2"),
             DataFormat.FLOAT32: np.dtype("<f4")}
_MAX_INT = {DataFormat.UINT8: 255, DataFormat.UINT16: 65535, DataFormat.FLOAT32: None}
_SHORT = {DataFormat.UINT8: "u8", DataFormat.UINT16: "u16", DataFormat.FLOAT32: "f32"}


class VoxelMapping:
    """Linear map stored value <-> application value on [lo, hi] (volume.py:73-99)."""

    __slots__ = ("lo", "hi")

    def __init__(self, lo: float, hi: float):
        lo, hi = float(lo), float(hi)
        if not (math.isfinite(lo) and math.isfinite(hi) and lo < hi):
            raise InvalidArgument(f"voxel mapping needs finite lo < hi, got [{lo}, {hi}]")
        self.lo, self.hi = lo, hi

    def __iter__(self):
        yield self.lo
        yield self.hi

    def __eq__(self, other):
        return isinstance(other, VoxelMapping) and (self.lo, self.hi) == (other.lo, other.hi)

    def __hash__(self):
        return hash((self.lo, self.hi))

    def __repr__(self):
        return f"VoxelMapping({self.lo}, {self.hi})"

    @classmethod
    def coerce(cls, value) -> "VoxelMapping":
        return value if isinstance(value, VoxelMapping) else cls(*value)


def quantize_scalar(value: float, fmt: DataFormat, mapping: VoxelMapping):
    """One application value -> stored value, the reference's rule.

    Same float64 operation sequence as ``quantize`` (volume.py:102-110):
    t = clip((v - lo)/(hi - lo), 0, 1); floor(t*max + 0.5) for the integer
    formats, round-to-nearest float32 otherwise.  Returns a numpy scalar of
    the storage dtype.
    """
    v = np.float64(value)
    if fmt is DataFormat.FLOAT32:
        return np.float32(v)
    t = np.clip((v - np.float64(mapping.lo)) / (np.float64(mapping.hi) - np.float64(mapping.lo)),
                0.0, 1.0)
    return fmt.dtype.type(np.floor(t * fmt.max_int + 0.5))


def dequantize_scalar(stored, fmt: DataFormat, mapping: VoxelMapping) -> float:
    """Stored value -> application value (volume.py:113-118)."""
    s = np.float64(stored)
    if fmt is DataFormat.FLOAT32:
        return float(s)
    return float(mapping.lo + (s / fmt.max_int) * (mapping.hi - mapping.lo))


def fill_bits(value: float, fmt: DataFormat, mapping: VoxelMapping) -> int:
    """``stored_bits(quantize_scalar(value, ...))`` without numpy scalars.

    Python floats are IEEE float64, so ``(v - lo) / (hi - lo)``, the clip,
    ``t * max + 0.5`` and ``floor`` round exactly as the numpy sequence of
    volume.py:102-110 does; float32 rounding goes through ``struct`` (round to
    nearest even, as ``np.float32``).  Non-finite inputs and float32
    overflow take the numpy path.  (The numpy scalar path cost ~15 us per
    FillRange call.)
    """
    v = float(value)
    if v - v == 0.0:  # finite
        if fmt is DataFormat.FLOAT32:
            try:
                return struct.unpack("<I", struct.pack("<f", v))[0]
            except OverflowError:
                pass
        else:
            lo, hi = float(mapping.lo), float(mapping.hi)
            t = (v - lo) / (hi - lo)
            t = 0.0 if t < 0.0 else (1.0 if t > 1.0 else t)
            return int(math.floor(t * fmt.max_int + 0.5))
    return stored_bits(quantize_scalar(value, fmt, mapping), fmt)


def stored_bits(value, fmt: DataFormat) -> int:
    """Bit pattern of a stored scalar, as the C ABI's fill entry point takes it."""
    arr = np.asarray([value], dtype=fmt.dtype)
    if fmt is DataFormat.FLOAT32:
        return int(arr.view("<u4")[0])
    return int(arr[0])


def _device(policy=None):
    import torch

    if not torch.cuda.is_available():
        raise DeviceFailure("no CUDA device is visible; the B200 path has no CPU fallback")
    policy = policy or get_execution_policy()
    idx = policy.device_index if policy.device_index is not None else torch.cuda.current_device()
    return torch.device("cuda", idx)


class DeviceBuffer:
    """A byte allocation in HBM; the device-resident ``ManagedBuffer``.

    ``migration_count`` stays 0: there is one residency (the reference's
    migrate() on a matching space is a no-op, managed.py:119-126).
    """

    def __init__(self, nbytes: int, device=None, zero: bool = True):
        import torch

        self.byte_length = int(nbytes)
        self.migration_count = 0
        dev = device if device is not None else _device()
        try:
            alloc = torch.zeros if zero else torch.empty
            self.tensor = alloc(max(self.byte_length, 1), dtype=torch.uint8, device=dev)
        except torch.OutOfMemoryError as e:
            raise AllocationFailure(f"device cannot hold {nbytes} bytes: {e}") from None

    @classmethod
    def wrap(cls, tensor) -> "DeviceBuffer":
        """Adopt an existing contiguous uint8 CUDA tensor (no copy)."""
        import torch

        if tensor.dtype != torch.uint8 or not tensor.is_cuda or not tensor.is_contiguous():
            raise InvalidArgument("DeviceBuffer.wrap needs a contiguous uint8 CUDA tensor")
        buf = cls.__new__(cls)
        buf.byte_length = int(tensor.numel())
        buf.migration_count = 0
        buf.tensor = tensor
        return buf

    def migrate(self) -> None:
        """No-op: the bytes are already in the only device space."""

    @property
    def array(self):
        return self.tensor[: self.byte_length]

    @property
    def device(self):
        return self.tensor.device

    def data_ptr(self) -> int:
        return int(self.tensor.data_ptr())

    def to_bytes(self) -> bytes:
        return self.array.cpu().numpy().tobytes()

    def __len__(self) -> int:
        return self.byte_length


class StructuredVolume:
    """Dense 3D cell grid in HBM (volume.py:121-234 semantics)."""

    def __init__(self, dims, fmt, cell_size=(1.0, 1.0, 1.0), mapping=(0.0, 1.0),
                 data: Optional[DeviceBuffer] = None):
        self.dims = ivec3(dims, "dims")
        if min(self.dims) < 1:
            raise InvalidArgument(f"dims must be >= 1 per axis, got {tuple(self.dims)}")
        self.format = fmt if isinstance(fmt, DataFormat) else DataFormat.parse(fmt)
        self.cell_size = fvec3(cell_size, "cell size")
        if min(self.cell_size) <= 0:
            raise InvalidArgument(f"cell size must be > 0 per axis, got {tuple(self.cell_size)}")
        self.mapping = VoxelMapping.coerce(mapping)
        nbytes = self.cell_count * self.format.bytes_per_cell
        if data is None:
            data = DeviceBuffer(nbytes)
        elif data.byte_length != nbytes:
            raise InvalidArgument(f"buffer holds {data.byte_length} bytes, volume needs {nbytes}")
        self.data = data

    # -- geometry ----------------------------------------------------------
    @property
    def cell_count(self) -> int:
        d = self.dims
        return d.x * d.y * d.z

    @property
    def world_extent(self) -> Vec3f:
        return Vec3f(*(n * c for n, c in zip(self.dims, self.cell_size)))

    @property
    def bounds(self) -> Box3i:
        return full_box(self.dims)

    @property
    def nbytes(self) -> int:
        return self.data.byte_length

    # -- storage -----------------------------------------------------------
    def array(self):
        """Device view of the stored values shaped (z, y, x)."""
        d = self.dims
        return self.data.array.view(self.format.torch_dtype).view(d.z, d.y, d.x)

    def data_ptr(self) -> int:
        return self.data.data_ptr()

    def to_numpy(self) -> np.ndarray:
        """Host copy of the stored values shaped (z, y, x)."""
        d = self.dims
        raw = self.data.array.cpu().numpy()
        return raw.view(self.format.dtype).reshape(d.z, d.y, d.x)

    def mapped_numpy(self) -> np.ndarray:
        """Host float64 application values (the reference's ``mapped_array``)."""
        s = self.to_numpy()
        if self.format is DataFormat.FLOAT32:
            return s.astype(np.float64)
        lo, hi = self.mapping
        return lo + (s.astype(np.float64) / self.format.max_int) * (hi - lo)

    def upload(self, host: np.ndarray, non_blocking: bool = False) -> None:
        """Copy a host array of the storage dtype (any shape with the right size) in."""
        import torch

        arr = np.ascontiguousarray(host)
        if arr.dtype != self.format.dtype or arr.size != self.cell_count:
            raise InvalidArgument(
                f"upload needs {self.cell_count} cells of {self.format.dtype}, "
                f"got {arr.size} of {arr.dtype}")
        src = torch.from_numpy(arr.reshape(-1).view(np.uint8))
        self.data.array.copy_(src, non_blocking=non_blocking)

    @classmethod
    def from_numpy(cls, host: np.ndarray, fmt=None, cell_size=(1.0, 1.0, 1.0),
                   mapping=(0.0, 1.0)) -> "StructuredVolume":
        """Volume from a host (z, y, x) array; format inferred from its dtype."""
        host = np.asarray(host)
        if host.ndim != 3:
            raise InvalidArgument("from_numpy needs a (z, y, x) array")
        if fmt is None:
            inv = {v: k for k, v in _NP_DTYPE.items()}
            key = host.dtype.newbyteorder("<") if host.dtype.byteorder == ">" else host.dtype
            if np.dtype(key) not in inv:
                raise InvalidArgument(f"no voxel format for dtype {host.dtype}")
            fmt = inv[np.dtype(key)]
        fmt = fmt if isinstance(fmt, DataFormat) else DataFormat.parse(fmt)
        nz, ny, nx = host.shape
        buf = DeviceBuffer(nx * ny * nz * fmt.bytes_per_cell, zero=False)
        v = cls((nx, ny, nz), fmt, cell_size, mapping, data=buf)
        v.upload(host.astype(fmt.dtype, copy=False))
        return v

    def fill_bytes(self, raw: bytes) -> None:
        import torch

        if len(raw) != self.data.byte_length:
            raise InvalidArgument(
                f"payload holds {len(raw)} bytes, volume needs {self.data.byte_length}")
        self.data.array.copy_(torch.frombuffer(bytearray(raw), dtype=torch.uint8))

    def copy(self) -> "StructuredVolume":
        out = StructuredVolume(self.dims, self.format, self.cell_size, self.mapping,
                               data=DeviceBuffer(self.nbytes, device=self.data.device, zero=False))
        out.data.array.copy_(self.data.array)
        return out

    def swap_storage(self, other: "StructuredVolume") -> None:
        """O(1) exchange of the device buffers of two same-shaped volumes."""
        self.data, other.data = other.data, self.data

    # -- single cells ------------------------------------------------------
    def _check_index(self, idx):
        idx = ivec3(idx, "cell index")
        if not all(0 <= i < n for i, n in zip(idx, self.dims)):
            raise IndexOutOfRange(f"index {tuple(idx)} outside dims {tuple(self.dims)}")
        return idx

    def get_value(self, idx) -> float:
        i = self._check_index(idx)
        stored = self.array()[i.z, i.y, i.x].cpu().numpy()
        return dequantize_scalar(stored, self.format, self.mapping)

    def set_value(self, idx, value: float) -> None:
        import torch

        i = self._check_index(idx)
        q = np.asarray([quantize_scalar(value, self.format, self.mapping)], dtype=self.format.dtype)
        self.array()[i.z, i.y, i.x] = torch.from_numpy(q)[0].to(self.data.device)

    def __repr__(self):
        d = self.dims
        return (f"StructuredVolume({d.x}x{d.y}x{d.z}, {self.format.short_name}, "
                f"range [{self.mapping.lo}, {self.mapping.hi}], {self.data.device})")


def create_structured_volume(dims, fmt, cell_size=(1.0, 1.0, 1.0), mapping=(0.0, 1.0)):
    """Zero-filled volume on the current CUDA device (volume.py:269-271)."""
    return StructuredVolume(dims, fmt, cell_size, mapping)


def require_same_layout(a: StructuredVolume, b: StructuredVolume) -> None:
    from .errors import DimsMismatch

    if tuple(a.dims) != tuple(b.dims) or a.format is not b.format or a.mapping != b.mapping:
        raise DimsMismatch(
            f"volumes differ: {tuple(a.dims)} {a.format.short_name} {a.mapping} vs "
            f"{tuple(b.dims)} {b.format.short_name} {b.mapping}")
    if a.data.device != b.data.device:
        raise DimsMismatch(f"volumes live on different devices: {a.data.device} vs {b.data.device}")


__all__ = [
    "DataFormat", "VoxelMapping", "StructuredVolume", "DeviceBuffer", "create_structured_volume",
    "quantize_scalar", "dequantize_scalar", "stored_bits", "fill_bits", "require_same_layout",
]
