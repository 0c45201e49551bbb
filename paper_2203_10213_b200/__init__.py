"""B200-native ApplyFilter for volkit-style structured volumes.

Drop-in for the reference's ApplyFilter hot path (arxiv 2203.10213, the
``vkt`` package at pkg/src/vkt): the names a caller of
``vkt.apply_filter`` / ``vkt.fill`` / ``vkt.fill_range`` uses are all here
with the same argument meaning and error classes, plus the north star's
``ApplyFilter(dst, src, filter, address_mode)``, ``Fill`` and ``FillRange``.
Volumes live in HBM; the arithmetic runs in hand-written sm_100a kernels
behind the C ABI in include/vkt_b200.h.  There is no CPU fallback.
"""

from . import errors
from .errors import (
    AllocationFailure,
    BadMagic,
    DeviceFailure,
    DimsMismatch,
    EmptyRange,
    EmptyVolume,
    NotASlab,
    IoFailure,
    NotSeekable,
    RangeOutOfBounds,
    SizeMismatch,
    TruncatedPayload,
    UnknownFormatCode,
    EvenKernelDims,
    IndexOutOfRange,
    InvalidArgument,
    VktError,
)
from .execution import (
    Device,
    ExecutionPolicy,
    FilterPath,
    effective_workers,
    get_execution_policy,
    hardware_concurrency,
    set_execution_policy,
    set_hardware_concurrency_override,
    timed,
    with_policy,
)
from .clahe import ClaheParams, brick_mappings, clahe_equalize
from .fill import Fill, FillRange, fill, fill_range
from .transforms import flip, resample
from .filters import (
    AddressMode,
    ApplyFilter,
    Filter,
    Kernel,
    apply_filter,
    apply_filter_host,
    box_kernel,
    chunk_planes,
    filter_path,
    gaussian_kernel,
    laplacian_kernel,
)
from .geom import Box3i, Vec3f, Vec3i, box3i, clip_box, full_box
from .volume import (
    DataFormat,
    DeviceBuffer,
    ManagedBuffer,
    StructuredVolume,
    VoxelMapping,
    create_structured_volume,
    dequantize_scalar,
    device_resident,
    emulated_device,
    quantize_scalar,
)
from .synthetic import synthetic_device, synthetic_host, synthetic_structured
from .io import (
    filter_file,
    load_raw,
    read_range,
    read_volume,
    volume_from_bytes,
    volume_to_bytes,
    write_range,
    write_volume,
)

from .benchmarks import run_benchmarks

__version__ = "0.2.0"

__all__ = [
    "AddressMode", "AllocationFailure", "ApplyFilter", "Box3i", "DataFormat", "Device",
    "DeviceBuffer", "DeviceFailure", "DimsMismatch", "EvenKernelDims", "ExecutionPolicy",
    "Fill", "FillRange", "Filter", "FilterPath", "IndexOutOfRange", "InvalidArgument", "Kernel",
    "StructuredVolume", "Vec3f", "Vec3i", "VktError", "VoxelMapping", "apply_filter",
    "apply_filter_host", "box3i",
    "box_kernel", "clip_box", "create_structured_volume", "dequantize_scalar", "errors", "fill",
    "fill_range", "filter_path", "full_box", "gaussian_kernel", "get_execution_policy",
    "laplacian_kernel", "quantize_scalar", "set_execution_policy", "synthetic_device",
    "synthetic_host", "synthetic_structured", "timed", "with_policy",
    "filter_file", "load_raw", "read_range", "read_volume", "volume_from_bytes", "volume_to_bytes",
    "write_range", "write_volume", "ClaheParams", "brick_mappings", "clahe_equalize",
    "flip", "resample", "ManagedBuffer", "emulated_device", "device_resident", "effective_workers",
    "hardware_concurrency", "set_hardware_concurrency_override", "run_benchmarks", "chunk_planes",
    "EmptyVolume", "NotASlab",
]
