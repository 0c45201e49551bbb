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
import threading
from enum import Enum
from typing import Optional

import struct
from contextlib import contextmanager

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


class DeviceSpace:
    """Capacity accounting of ``ManagedBuffer`` bytes resident in HBM.

    The reference's ``emulated_device`` arena (managed.py:31-59) has an
    optional capacity so allocation failure is observable; here the arena is
    the B200's HBM and the same accounting applies to the managed volumes
    placed there (``AllocationFailure`` past the capacity, or on a real CUDA
    out-of-memory).
    """

    def __init__(self, capacity_bytes: Optional[int] = None):
        self.capacity_bytes = capacity_bytes
        self.used_bytes = 0
        self._lock = threading.Lock()

    def set_capacity(self, capacity_bytes: Optional[int]) -> None:
        with self._lock:
            self.capacity_bytes = capacity_bytes

    def reserve(self, nbytes: int) -> None:
        with self._lock:
            if self.capacity_bytes is not None and self.used_bytes + nbytes > self.capacity_bytes:
                raise AllocationFailure(
                    f"device cannot hold {nbytes} bytes ({self.used_bytes}/{self.capacity_bytes} in use)")
            self.used_bytes += nbytes

    def release(self, nbytes: int) -> None:
        with self._lock:
            self.used_bytes -= nbytes


#: Process-wide HBM accounting for managed volumes (the reference's name).
emulated_device = DeviceSpace()


def _alloc_device(nbytes: int, dev, zero: bool):
    import torch

    try:
        alloc = torch.zeros if zero else torch.empty
        return alloc(max(nbytes, 1), dtype=torch.uint8, device=dev)
    except torch.OutOfMemoryError as e:
        raise AllocationFailure(f"device cannot hold {nbytes} bytes: {e}") from None


def _alloc_host(nbytes: int, zero: bool):
    """Page-locked host bytes: the device reads and writes them directly
    (unified addressing), and copies to and from HBM run at full PCIe rate."""
    import torch

    if not torch.cuda.is_available():
        raise DeviceFailure("no CUDA device is visible; the B200 path has no CPU fallback")
    t = torch.empty(max(nbytes, 1), dtype=torch.uint8, pin_memory=True)
    if zero:
        t.zero_()
    return t


class _Storage:
    """Bytes of a volume in one residency: ``tensor`` is a uint8 torch tensor
    in HBM or in page-locked host memory."""

    byte_length: int
    migration_count: int
    tensor: "object"

    @property
    def on_host(self) -> bool:
        return not self.tensor.is_cuda

    @property
    def residency(self):
        from .execution import Device

        return Device.CPU if self.on_host else Device.CUDA

    @property
    def raw(self):
        """The bytes as a torch tensor (host or device)."""
        return self.tensor[: self.byte_length]

    @property
    def array(self):
        """The resident bytes: a numpy view on the host, a torch view in HBM."""
        if self.on_host:
            return self.tensor[: self.byte_length].numpy()
        return self.tensor[: self.byte_length]

    @property
    def device(self):
        return self.tensor.device

    def data_ptr(self) -> int:
        return int(self.tensor.data_ptr())

    def to_bytes(self) -> bytes:
        raw = self.raw
        return (raw.numpy() if self.on_host else raw.cpu().numpy()).tobytes()

    def empty_like(self) -> "_Storage":
        """Uninitialized bytes of the same length and residency."""
        out = _Storage.__new__(type(self))
        out.byte_length = self.byte_length
        out.migration_count = 0
        out.tensor = (_alloc_host(self.byte_length, False) if self.on_host
                      else _alloc_device(self.byte_length, self.tensor.device, False))
        if isinstance(out, ManagedBuffer):
            if not out.on_host:
                emulated_device.reserve(out.byte_length)
            out._init_accounting()
        return out

    def __len__(self) -> int:
        return self.byte_length


class DeviceBuffer(_Storage):
    """A byte allocation in HBM: the native API's fixed-residency buffer.

    ``migration_count`` stays 0: its residency never changes (the reference's
    migrate() on a matching space is a no-op, managed.py:119-126).
    """

    def __init__(self, nbytes: int, device=None, zero: bool = True):
        self.byte_length = int(nbytes)
        self.migration_count = 0
        self.tensor = _alloc_device(self.byte_length, device if device is not None else _device(), zero)

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
        """No-op: the bytes stay in HBM."""


def _managed_policy():
    from .execution import explicit_policy

    return explicit_policy()


class ManagedBuffer(_Storage):
    """The reference's managed byte buffer (managed.py:97-154): resident in
    exactly one space, the one the calling thread's policy selects.

    ``Device.CPU`` keeps the bytes in page-locked host memory (``array`` is a
    numpy view); ``Device.EMULATED_DEVICE`` / ``Device.CUDA`` in HBM.  With
    no policy set on the thread the reference's default applies: the host.
    ``migrate()`` moves them when the policy's space differs and counts the
    move in ``migration_count``; algorithms call it before touching the data.
    """

    def __init__(self, initial, device=None):
        if isinstance(initial, (int, np.integer)):
            self.byte_length = int(initial)
            host = None
        else:
            host = np.frombuffer(bytes(initial), dtype=np.uint8)
            self.byte_length = int(host.size)
        self.migration_count = 0
        policy = _managed_policy()
        if policy is None or policy.device.on_host:
            self.tensor = _alloc_host(self.byte_length, host is None)
        else:
            emulated_device.reserve(self.byte_length)
            try:
                self.tensor = _alloc_device(self.byte_length, device if device is not None else _device(policy),
                                            host is None)
            except BaseException:
                emulated_device.release(self.byte_length)
                raise
        self._init_accounting()
        if host is not None and host.size:
            self.raw.copy_(__import__("torch").from_numpy(host.copy()))

    def _init_accounting(self) -> None:
        self._charged = 0 if self.on_host else self.byte_length
        self._lock = threading.Lock()

    def migrate(self) -> None:
        """Move the bytes to the current policy's space if they are elsewhere."""
        from .execution import debug

        policy = _managed_policy()
        want_host = policy is None or policy.device.on_host
        with self._lock:
            if want_host == self.on_host:
                return
            if want_host:
                dst = _alloc_host(self.byte_length, False)
                dst[: self.byte_length].copy_(self.raw)  # synchronous D2H
                emulated_device.release(self._charged)
                self._charged = 0
            else:
                emulated_device.reserve(self.byte_length)
                try:
                    dst = _alloc_device(self.byte_length, _device(policy), False)
                except BaseException:
                    emulated_device.release(self.byte_length)
                    raise
                dst[: self.byte_length].copy_(self.raw)
                self._charged = self.byte_length
            debug(f"migrate {self.byte_length} bytes {'device -> host' if want_host else 'host -> device'}")
            self.tensor = dst
            self.migration_count += 1

    def __del__(self):
        try:
            if self._charged:
                emulated_device.release(self._charged)
        except Exception:
            pass


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
            data = self._new_storage(nbytes)
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
    @property
    def on_host(self) -> bool:
        """True when the bytes live in page-locked host memory (``Device.CPU``)."""
        return self.data.on_host

    def array(self):
        """Stored values shaped (z, y, x), after migrating to the policy's
        space (volume.py:172-177): a numpy view for host-resident volumes, a
        torch CUDA view for volumes in HBM."""
        self.data.migrate()
        d = self.dims
        if self.data.on_host:
            return self.data.array.view(self.format.dtype).reshape(d.z, d.y, d.x)
        return self.data.array.view(self.format.torch_dtype).view(d.z, d.y, d.x)

    def mapped_array(self) -> np.ndarray:
        """Host float64 application values shaped (z, y, x) (volume.py:179-181):
        dequantize in the reference's float64 operation order (volume.py:113-118)."""
        s = self.to_numpy()
        if self.format is DataFormat.FLOAT32:
            return np.asarray(s, dtype=np.float64)
        lo, hi = self.mapping
        return lo + (np.asarray(s, dtype=np.float64) / self.format.max_int) * (hi - lo)

    #: former name of ``mapped_array``
    mapped_numpy = mapped_array

    def normalized_array(self) -> np.ndarray:
        """Mapping-normalized values in [0, 1] (volume.py:183-186)."""
        m = self.mapped_array()
        lo, hi = self.mapping
        return np.clip((m - lo) / (hi - lo), 0.0, 1.0)

    def data_ptr(self) -> int:
        return self.data.data_ptr()

    def to_numpy(self) -> np.ndarray:
        """Host copy of the stored values shaped (z, y, x)."""
        d = self.dims
        raw = self.data.raw
        host = raw.numpy().copy() if self.data.on_host else raw.cpu().numpy()
        return host.view(self.format.dtype).reshape(d.z, d.y, d.x)

    def upload(self, host: np.ndarray, non_blocking: bool = False) -> None:
        """Copy a host array of the storage dtype (any shape with the right size) in."""
        import torch

        arr = np.ascontiguousarray(host)
        if arr.dtype != self.format.dtype or arr.size != self.cell_count:
            raise InvalidArgument(
                f"upload needs {self.cell_count} cells of {self.format.dtype}, "
                f"got {arr.size} of {arr.dtype}")
        src = torch.from_numpy(arr.reshape(-1).view(np.uint8))
        self.data.raw.copy_(src, non_blocking=non_blocking and not self.data.on_host)

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
        v = cls((nx, ny, nz), fmt, cell_size, mapping, data=cls._new_storage(nx * ny * nz * fmt.bytes_per_cell, zero=False))
        v.upload(host.astype(fmt.dtype, copy=False))
        return v

    @classmethod
    def _new_storage(cls, nbytes: int, zero: bool = True):
        """Default storage of new volumes: HBM (the façade in ``.vkt`` overrides
        this with a policy-following ``ManagedBuffer``)."""
        return DeviceBuffer(nbytes, zero=zero)

    def fill_bytes(self, raw: bytes) -> None:
        import torch

        if len(raw) != self.data.byte_length:
            raise InvalidArgument(
                f"payload holds {len(raw)} bytes, volume needs {self.data.byte_length}")
        self.data.migrate()
        self.data.raw.copy_(torch.frombuffer(bytearray(raw), dtype=torch.uint8))

    def copy(self) -> "StructuredVolume":
        self.data.migrate()
        out = type(self)(self.dims, self.format, self.cell_size, self.mapping, data=self.data.empty_like())
        out.data.raw.copy_(self.data.raw)
        return out

    def swap_storage(self, other: "StructuredVolume") -> None:
        """O(1) exchange of the bytes of two same-shaped volumes (the buffer
        objects, and their migration counts, stay with their volumes)."""
        a, b = self.data, other.data
        if type(a) is type(b):
            a.tensor, b.tensor = b.tensor, a.tensor
            if isinstance(a, ManagedBuffer):
                a._charged, b._charged = b._charged, a._charged
        else:
            self.data, other.data = b, a

    # -- single cells ------------------------------------------------------
    def _check_index(self, idx):
        idx = ivec3(idx, "cell index")
        if not all(0 <= i < n for i, n in zip(idx, self.dims)):
            raise IndexOutOfRange(f"index {tuple(idx)} outside dims {tuple(self.dims)}")
        return idx

    def get_value(self, idx) -> float:
        i = self._check_index(idx)
        cell = self.array()[i.z, i.y, i.x]
        stored = cell if self.data.on_host else cell.cpu().numpy()
        return dequantize_scalar(stored, self.format, self.mapping)

    def set_value(self, idx, value: float) -> None:
        import torch

        i = self._check_index(idx)
        q = np.asarray([quantize_scalar(value, self.format, self.mapping)], dtype=self.format.dtype)
        arr = self.array()
        if self.data.on_host:
            arr[i.z, i.y, i.x] = q[0]
        else:
            arr[i.z, i.y, i.x] = torch.from_numpy(q)[0].to(self.data.device)

    def __repr__(self):
        d = self.dims
        return (f"StructuredVolume({d.x}x{d.y}x{d.z}, {self.format.short_name}, "
                f"range [{self.mapping.lo}, {self.mapping.hi}], {self.data.device})")


@contextmanager
def device_resident(volume: "StructuredVolume", write_back: bool = True):
    """Yield a volume whose bytes are in HBM for a device algorithm: the
    volume itself, or for a host-resident (``Device.CPU``) volume a device
    copy whose result is copied back (``write_back``) before returning."""
    import torch

    volume.data.migrate()
    if not volume.data.on_host:
        yield volume
        return
    dev = StructuredVolume(volume.dims, volume.format, volume.cell_size, volume.mapping,
                           data=DeviceBuffer(volume.nbytes, zero=False))
    dev.data.raw.copy_(volume.data.raw)
    yield dev
    if write_back:
        volume.data.raw.copy_(dev.data.raw)  # synchronous D2H into the pinned bytes
    torch.cuda.current_stream().synchronize()


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
    "DataFormat", "VoxelMapping", "StructuredVolume", "DeviceBuffer", "ManagedBuffer", "DeviceSpace",
    "emulated_device", "device_resident", "create_structured_volume",
    "quantize_scalar", "dequantize_scalar", "stored_bits", "fill_bits", "require_same_layout",
]
