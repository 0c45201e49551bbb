"""The reference's error module (pkg/src/vkt/errors.py): the same classes,
re-exported from the package's error contract."""

from ..errors import *  # noqa: F401,F403
from ..errors import (  # noqa: F401
    AllocationFailure, BadMagic, DeviceFailure, DimsMismatch, EmptyRange, EmptyVolume,
    EvenKernelDims, IndexOutOfRange, InvalidArgument, IoFailure, NotASlab, NotSeekable,
    RangeOutOfBounds, SizeMismatch, TruncatedPayload, UnknownFormatCode, VktError,
)
