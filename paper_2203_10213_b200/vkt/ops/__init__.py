"""``vkt.ops`` (pkg/src/vkt/ops/__init__.py), restricted to the ApplyFilter path."""

from .core import fill, fill_range  # noqa: F401
from .filters import ClaheParams, Kernel, apply_filter, box_kernel, clahe_equalize, gaussian_kernel  # noqa: F401
