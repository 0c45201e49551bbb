"""``vkt.ops.filters`` (pkg/src/vkt/ops/filters.py): kernels, ApplyFilter and
CLAHE, B200-backed.  ``_clip_counts`` is the clip rule the reference's own
tests import (tests/test_ops_filter.py:10)."""

from ...clahe import ClaheParams, _axis_edges, _blend_coords, _clip_counts, brick_mappings, clahe_equalize  # noqa: F401
from ...filters import Kernel, apply_filter, box_kernel, gaussian_kernel  # noqa: F401
