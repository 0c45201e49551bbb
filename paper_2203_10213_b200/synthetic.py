"""Synthetic input volumes.

``synthetic_structured`` reproduces the reference generator bit-for-bit
(pkg/src/vkt/bench.py:38-48: numpy ``default_rng(seed)``; u8/u16 uniform
integers over [0, max], f32 ``rng.random`` in [0, 1)) on the host and uploads
it — used for parity runs.  ``synthetic_device`` draws the same distributions
from a counter-based hash of the global cell index directly in HBM
(``vkt_fill_synthetic``), so a z-slab shard generates exactly the planes of the
unsharded volume without any host work — used for throughput runs.
"""

from __future__ import annotations

import numpy as np

from . import _capi
from .volume import DataFormat, DeviceBuffer, StructuredVolume


def synthetic_host(size, fmt: DataFormat = DataFormat.UINT8, seed: int = 7) -> np.ndarray:
    """Host (z, y, x) array with the reference generator's exact values."""
    if isinstance(size, int):
        size = (size, size, size)
    nx, ny, nz = size
    rng = np.random.default_rng(seed)
    if fmt is DataFormat.FLOAT32:
        return rng.random((nz, ny, nx), dtype=np.float32)
    info = np.iinfo(fmt.dtype)
    return rng.integers(0, info.max + 1, size=(nz, ny, nx), dtype=fmt.dtype)


def synthetic_structured(size, fmt: DataFormat = DataFormat.UINT8, seed: int = 7) -> StructuredVolume:
    """Device volume holding ``synthetic_host(size, fmt, seed)``."""
    return StructuredVolume.from_numpy(synthetic_host(size, fmt, seed), fmt)


def synthetic_device(dims, fmt: DataFormat, seed: int = 7, *, z_offset: int = 0,
                     local_nz: int | None = None, device=None) -> StructuredVolume:
    """Hash-generated volume (or the z-slab [z_offset, z_offset+local_nz) of one)."""
    import torch

    nx, ny, nz = dims
    lnz = nz - z_offset if local_nz is None else local_nz
    buf = DeviceBuffer(nx * ny * lnz * fmt.bytes_per_cell, device=device, zero=False)
    vol = StructuredVolume((nx, ny, lnz), fmt, data=buf)
    stream = torch.cuda.current_stream(buf.device)
    _capi.check(_capi.load().vkt_fill_synthetic(
        vol.data_ptr(), _capi.int3((nx, ny, lnz)), fmt.value, int(seed), int(z_offset),
        int(stream.cuda_stream)))
    return vol
