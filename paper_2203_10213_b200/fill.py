"""Fill / FillRange: the input builders of the ApplyFilter path.

Reference: ``fill_range(volume, roi, value)`` clips the roi to the volume,
returns on an empty roi, quantizes the scalar once and slice-assigns it
(pkg/src/vkt/ops/core.py:39-55); ``fill`` is the full box (core.py:65-66).
Here the scalar is quantized once on the host with the same float64 rule
(volume.py:102-110) and the device performs a pure box store of that bit
pattern (``vkt_fill_box``), so the result is bit-exact by construction.  The
store goes to HBM, or for host-resident volumes into their page-locked bytes.
"""

from __future__ import annotations

from . import _capi
from .execution import timed
from .geom import clip_box, coerce_box
from .volume import StructuredVolume, fill_bits


@timed("FillRange")
def fill_range(volume: StructuredVolume, roi, value: float) -> None:
    """Set every cell of ``roi`` ∩ bounds to ``value`` (asynchronous)."""
    import torch

    box = clip_box(coerce_box(roi), volume.bounds)
    if box.is_empty:
        return
    bits = fill_bits(value, volume.format, volume.mapping)
    volume.data.migrate()
    # HBM volumes: asynchronous on the volume's current stream.  Host-resident
    # (Device.CPU) volumes: the same kernel stores straight into the
    # page-locked bytes (unified addressing) and the call waits for it, since
    # their numpy views are read right away.
    host = volume.on_host
    stream = torch.cuda.current_stream() if host else torch.cuda.current_stream(volume.data.device)
    _capi.check(_capi.load().vkt_fill_box(
        volume.data_ptr(), _capi.int3(volume.dims), volume.format.value,
        _capi.int3(box.lower), _capi.int3(box.upper), bits, int(stream.cuda_stream)))
    if host:
        stream.synchronize()


def fill(volume: StructuredVolume, value: float) -> None:
    """Whole-volume fill (core.py:65-66)."""
    fill_range(volume, volume.bounds, value)


#: North-star spellings.
FillRange = fill_range
Fill = fill
