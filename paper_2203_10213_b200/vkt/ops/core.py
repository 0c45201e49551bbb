"""``vkt.ops.core`` (pkg/src/vkt/ops/core.py), the Fill / FillRange helpers."""

from ...fill import fill, fill_range  # noqa: F401
from ...transforms import resample  # noqa: F401
