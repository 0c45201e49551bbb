"""Error contract of the drop-in.

The reference identifies failures by exception class name across process and
language boundaries (``VktError.name``, pkg/src/vkt/errors.py:9-14).  The
classes the ApplyFilter / Fill path can raise keep those names; the C ABI's
status codes map onto them through ``vkt_status_name`` (include/vkt_b200.h).
"""

from __future__ import annotations


class VktError(Exception):
    """Root of every error this package raises; ``name`` is the class name."""

    @property
    def name(self) -> str:
        return self.__class__.__name__


class InvalidArgument(VktError):
    """A documented precondition does not hold (errors.py:17)."""


class IndexOutOfRange(VktError):
    """Cell index outside the volume (errors.py:21)."""


class AllocationFailure(VktError):
    """Device memory cannot hold the requested bytes (errors.py:25)."""


class EvenKernelDims(VktError):
    """Kernel extents must be odd on every axis (errors.py:53)."""


class DimsMismatch(VktError):
    """Operand volumes disagree in dimensions, format or mapping (errors.py:49)."""


class EmptyRange(VktError):
    """The region of interest selects no cells (errors.py:37)."""


class RangeOutOfBounds(VktError):
    """The region of interest extends past the volume bounds (errors.py:41)."""


class NotASlab(VktError):
    """A Delete region is not a full-extent slab (errors.py:45).  Kept so
    reference callers that import it run unchanged; not raised on this path."""


class EmptyVolume(VktError):
    """A volume with zero cells (errors.py:33); kept for the same reason."""


class BadMagic(VktError):
    """The stream does not start with VKTVOL01 (errors.py:57)."""


class TruncatedPayload(VktError):
    """The stream ends before the header-implied byte count (errors.py:61)."""


class UnknownFormatCode(VktError):
    """Unrecognised data-format or volume-type code (errors.py:65)."""


class IoFailure(VktError):
    """A read, write or flush failed (errors.py:69)."""


class SizeMismatch(VktError):
    """Raw payload length disagrees with the requested geometry (errors.py:73)."""


class NotSeekable(VktError):
    """Range I/O needs a seekable source (errors.py:77)."""


class DeviceFailure(VktError):
    """The CUDA runtime reported an error, or no CUDA device / library exists.

    New in this package: the reference has no accelerator (its "device" is
    an emulated arena, managed.py:31-59), so it never raises this.
    """


_BY_NAME = {
    cls.__name__: cls
    for cls in (InvalidArgument, IndexOutOfRange, AllocationFailure, EvenKernelDims,
                DimsMismatch, DeviceFailure, EmptyRange, RangeOutOfBounds, NotASlab, EmptyVolume, BadMagic,
                TruncatedPayload, UnknownFormatCode, IoFailure, SizeMismatch, NotSeekable)
}


def from_status_name(name: str, detail: str) -> VktError:
    """Exception instance for a C-ABI status name (``vkt_status_name``)."""
    return _BY_NAME.get(name, DeviceFailure)(detail)
