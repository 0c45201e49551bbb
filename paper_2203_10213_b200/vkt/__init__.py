"""The reference's ``vkt`` namespace on the ApplyFilter path, B200-backed.

``import paper_2203_10213_b200.vkt as vkt`` gives a caller of the reference
(pkg/src/vkt/__init__.py) the names its ApplyFilter / Fill code uses, with the
reference's semantics:

* volumes are backed by a ``ManagedBuffer`` whose residency follows the
  calling thread's ``ExecutionPolicy`` (managed.py:97-154) — by default the
  host, where ``array()`` is a writable numpy view exactly as in the
  reference; ``Device.EMULATED_DEVICE`` places the bytes in HBM;
* every algorithm computes on the B200 whatever the residency (a host volume
  is streamed through HBM; there is no CPU compute path);
* errors, policies, ``effective_workers``, ``emulated_device`` capacity
  accounting and ``run_benchmarks`` keep their names and meaning.

The native package (``paper_2203_10213_b200``) is the device-first API the
benchmark uses: its volumes live in HBM from the start.  Both share the same
kernels, policies and error classes; this module only changes the default
storage of new volumes and the default policy.

Not on the path and not provided: hierarchical volumes, rendering, analysis
(aggregates / histograms), crop and arithmetic.
"""

from __future__ import annotations

from dataclasses import dataclass, replace

from .. import errors
from ..benchmarks import run_benchmarks
from ..clahe import ClaheParams, clahe_equalize
from ..errors import VktError
from ..execution import Device, FilterPath
from ..execution import ExecutionPolicy as _NativePolicy
from ..execution import (
    effective_workers,
    explicit_policy,
    hardware_concurrency,
    set_execution_policy,
    set_hardware_concurrency_override,
    timed,
)
from ..fill import fill, fill_range
from ..filters import Kernel, apply_filter, box_kernel, gaussian_kernel
from ..geom import Box3i, Vec3f, Vec3i, box3i, full_box
from ..io import read_range, read_volume, volume_from_bytes, volume_to_bytes, write_range, write_volume
from ..synthetic import synthetic_host
from ..transforms import flip, resample
from ..volume import DataFormat, ManagedBuffer, VoxelMapping, emulated_device
from ..volume import StructuredVolume as _DeviceVolume


@dataclass(frozen=True)
class ExecutionPolicy(_NativePolicy):
    """The reference's policy (execution.py:37-51): default device CPU."""

    device: Device = Device.CPU


_DEFAULT = ExecutionPolicy()


def get_execution_policy() -> _NativePolicy:
    """Policy last set on this thread, or the reference's CPU default."""
    return explicit_policy() or _DEFAULT


def with_policy(**changes) -> _NativePolicy:
    """Copy of the current policy with fields replaced, not installed
    (execution.py:199-201)."""
    return replace(get_execution_policy(), **changes)


class StructuredVolume(_DeviceVolume):
    """``StructuredVolume`` (volume.py:121-234) whose bytes live in a
    policy-following ``ManagedBuffer`` (host by default)."""

    @classmethod
    def _new_storage(cls, nbytes: int, zero: bool = True):
        return ManagedBuffer(nbytes)


def create_structured_volume(dims, fmt, cell_size=(1.0, 1.0, 1.0), mapping=(0.0, 1.0)) -> StructuredVolume:
    """Zero-filled volume in the policy's space (volume.py:269-271)."""
    return StructuredVolume(dims, fmt, cell_size, mapping)


def synthetic_structured(size: int, fmt: DataFormat = DataFormat.UINT8, seed: int = 7) -> StructuredVolume:
    """The reference generator's cube (bench.py:38-48) in the policy's space."""
    return StructuredVolume.from_numpy(synthetic_host(size, fmt, seed), fmt)


__all__ = [
    "Box3i", "ClaheParams", "DataFormat", "Device", "ExecutionPolicy", "FilterPath", "Kernel",
    "ManagedBuffer", "StructuredVolume", "Vec3f", "Vec3i", "VktError", "VoxelMapping",
    "apply_filter", "box3i", "box_kernel", "clahe_equalize", "create_structured_volume",
    "effective_workers", "emulated_device", "errors", "fill", "fill_range", "flip", "full_box",
    "gaussian_kernel", "get_execution_policy", "hardware_concurrency", "read_range",
    "read_volume", "resample", "run_benchmarks", "set_execution_policy",
    "set_hardware_concurrency_override", "synthetic_structured", "timed", "volume_from_bytes",
    "volume_to_bytes", "with_policy", "write_range", "write_volume",
]
