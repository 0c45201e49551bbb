"""CLAHE-3D on the B200 — the paper's case study.

Reference: ``clahe_equalize`` / ``brick_mappings`` / ``ClaheParams``
(pkg/src/vkt/ops/filters.py:98-245).  The volume is split into bricks; each
brick's histogram of normalized values is clipped and turned into a cdf
mapping, and every cell blends the mappings of its 8 nearest brick centers.

Division of work (bit-identical to the reference):
  * device: per-brick histograms (``vkt_clahe_histograms``; integer atomics,
    exact) and the per-cell blend + quantize (``vkt_clahe_blend``; IEEE
    float64 in numpy's operation order);
  * host: the tiny per-axis tables (brick edges, blend coordinates) and the
    per-brick clip + cdf, with the same numpy operations as the reference.
"""

from __future__ import annotations

import ctypes
import math
from dataclasses import dataclass

import numpy as np

from . import _capi
from .errors import InvalidArgument
from .execution import timed
from .geom import Vec3i, ivec3
from .volume import DataFormat, StructuredVolume, device_resident


@dataclass
class ClaheParams:
    """Brick grid, histogram resolution and contrast clip (filters.py:101-115).

    ``clip_limit`` is a multiple of the uniform bin height; ``math.inf``
    disables clipping.
    """

    brick_counts: Vec3i
    num_bins: int = 256
    clip_limit: float = math.inf

    def __post_init__(self):
        self.brick_counts = ivec3(self.brick_counts, "brick counts")


class ClaheArgs(ctypes.Structure):
    _fields_ = [
        ("src", ctypes.c_void_p), ("dst", ctypes.c_void_p), ("dims", _capi.Int3),
        ("format", ctypes.c_int32), ("map_lo", ctypes.c_double), ("map_hi", ctypes.c_double),
        ("bricks", _capi.Int3), ("num_bins", ctypes.c_int32), ("bin_lut", ctypes.c_void_p),
        ("edges", ctypes.c_void_p), ("hist", ctypes.c_void_p), ("mappings", ctypes.c_void_p),
        ("blend_lo", ctypes.c_void_p), ("blend_w", ctypes.c_void_p),
    ]


def _lib():
    lib = _capi.load()
    if not getattr(lib, "_clahe_typed", False):
        lib.vkt_clahe_histograms.argtypes = [ctypes.POINTER(ClaheArgs), ctypes.c_void_p]
        lib.vkt_clahe_histograms.restype = ctypes.c_int
        lib.vkt_clahe_blend.argtypes = [ctypes.POINTER(ClaheArgs), ctypes.c_void_p]
        lib.vkt_clahe_blend.restype = ctypes.c_int
        lib._clahe_typed = True
    return lib


# -- host tables ---------------------------------------------------------------
# Restated from the reference's definitions (ops/filters.py:117-147); integer
# results are identical by construction and the float64 blend weights use the
# same operations (an exact halving for the centres, one subtract / divide /
# clip per cell), so the tables are bit-identical (tests/test_clahe.py).

def _axis_edges(extent: int, count: int) -> np.ndarray:
    """Brick boundaries of ``count`` bricks over ``extent`` cells; the first
    ``extent % count`` bricks are one cell thicker (filters.py:118-122)."""
    i = np.arange(count + 1, dtype=np.int64)
    return i * (extent // count) + np.minimum(i, extent % count)


def _clip_counts(hist: np.ndarray, limit: int) -> np.ndarray:
    """Clip every bin at ``limit`` once and hand the clipped total back in
    equal shares, the indivisible rest one count each to the lowest bins
    (filters.py:124-132)."""
    over = hist - limit
    excess = int(over[over > 0].sum())
    out = np.minimum(hist, limit) + excess // hist.size
    out[: excess % hist.size] += 1
    return out


def _blend_coords(extent: int, edges: np.ndarray):
    """For each cell centre along one axis: the lower of the two brick centres
    it blends between and its weight toward the upper one, clamped to the
    outermost bricks (filters.py:135-147)."""
    nb = len(edges) - 1
    if nb == 1:
        return np.zeros(extent, dtype=np.int64), np.zeros(extent)
    mid = (edges[1:] + edges[:-1]) / 2.0
    pos = np.arange(extent, dtype=np.float64) + 0.5
    lower = np.clip(np.digitize(pos, mid) - 1, 0, nb - 2)
    span = mid[lower + 1] - mid[lower]
    return lower, np.clip((pos - mid[lower]) / span, 0.0, 1.0)


def _validate(volume: StructuredVolume, params: ClaheParams) -> None:
    """filters.py:150-160."""
    if params.num_bins < 2:
        raise InvalidArgument(f"CLAHE needs num_bins >= 2, got {params.num_bins}")
    c = params.brick_counts
    if min(c) < 1 or any(c[a] > volume.dims[a] for a in range(3)):
        raise InvalidArgument(f"brick counts {tuple(c)} invalid for dims {tuple(volume.dims)}")
    if not (params.clip_limit >= 1.0):
        raise InvalidArgument(f"clip limit must be >= 1 (or inf), got {params.clip_limit}")


def _bin_lut(fmt: DataFormat, lo: float, hi: float, nbins: int):
    """Stored value -> bin for the integer formats, numpy's float64 rule:
    t = clip((dequantize(s) - lo)/(hi - lo), 0, 1); min(nbins-1, floor(t*nbins))
    (volume.py:113-118, 183-186; filters.py:172-173)."""
    if fmt is DataFormat.FLOAT32:
        return None
    s = np.arange(fmt.max_int + 1, dtype=np.float64)
    m = lo + (s / fmt.max_int) * (hi - lo)
    t = np.clip((m - lo) / (hi - lo), 0.0, 1.0)
    return np.minimum(nbins - 1, np.floor(t * nbins)).astype(np.int32)


def _device(arr: np.ndarray, dev):
    import torch

    return torch.from_numpy(np.ascontiguousarray(arr)).to(dev)


def _args(volume: StructuredVolume, params: ClaheParams, dev, keep: list) -> ClaheArgs:
    c = params.brick_counts
    d = volume.dims
    edges = np.concatenate([_axis_edges(d.x, c.x), _axis_edges(d.y, c.y),
                            _axis_edges(d.z, c.z)]).astype(np.int32)
    lut = _bin_lut(volume.format, volume.mapping.lo, volume.mapping.hi, params.num_bins)
    a = ClaheArgs()
    a.src = volume.data_ptr()
    a.dst = volume.data_ptr()
    a.dims = _capi.int3(d)
    a.format = volume.format.value
    a.map_lo, a.map_hi = volume.mapping.lo, volume.mapping.hi
    a.bricks = _capi.int3(c)
    a.num_bins = int(params.num_bins)
    t_edges = _device(edges, dev)
    keep.append(t_edges)
    a.edges = t_edges.data_ptr()
    if lut is not None:
        t_lut = _device(lut, dev)
        keep.append(t_lut)
        a.bin_lut = t_lut.data_ptr()
    return a


def _stream(dev) -> ctypes.c_void_p:
    import torch

    return ctypes.c_void_p(int(torch.cuda.current_stream(dev).cuda_stream))


def _histograms(volume: StructuredVolume, params: ClaheParams, keep: list) -> tuple[np.ndarray, ClaheArgs]:
    import torch

    dev = volume.data.device
    a = _args(volume, params, dev, keep)
    c = params.brick_counts
    hist = torch.zeros(c.x * c.y * c.z * params.num_bins, dtype=torch.int32, device=dev)
    keep.append(hist)
    a.hist = hist.data_ptr()
    _capi.check(_lib().vkt_clahe_histograms(ctypes.byref(a), _stream(dev)))
    h = hist.cpu().numpy().view(np.uint32).astype(np.int64).reshape(c.z, c.y, c.x, params.num_bins)
    return h, a


def _mappings_from_hist(h: np.ndarray, volume: StructuredVolume, params: ClaheParams) -> np.ndarray:
    """Clip + cdf / n_cells per brick, as brick_mappings does (filters.py:188-201),
    for all bricks at once: the same integer clip (_clip_counts) and the same
    float64 cumsum / n_cells per element as the per-brick loop."""
    c = params.brick_counts
    d = volume.dims
    ex, ey, ez = _axis_edges(d.x, c.x), _axis_edges(d.y, c.y), _axis_edges(d.z, c.z)
    nb = params.num_bins
    n_cells = (np.diff(ez)[:, None, None] * np.diff(ey)[None, :, None] * np.diff(ex)[None, None, :]).astype(np.int64)
    hist = h.astype(np.int64)
    if math.isfinite(params.clip_limit):
        # limit = max(1, floor(clip * n_cells / nb + 0.5)) in float64, per brick
        limit = np.maximum(1, np.floor(params.clip_limit * n_cells.astype(np.float64) / nb + 0.5)).astype(np.int64)
        lim = limit[..., None]
        excess = np.maximum(hist - lim, 0).sum(axis=-1)
        share, rem = np.divmod(excess, nb)
        hist = np.minimum(hist, lim) + share[..., None] + (np.arange(nb) < rem[..., None])
    return np.cumsum(hist, axis=-1) / n_cells.astype(np.float64)[..., None]


def brick_mappings(volume: StructuredVolume, params: ClaheParams) -> np.ndarray:
    """Per-brick equalization maps, shape (bz, by, bx, num_bins) (filters.py:163-201)."""
    _validate(volume, params)
    keep: list = []
    with device_resident(volume, write_back=False) as v:
        h, _ = _histograms(v, params, keep)
        return _mappings_from_hist(h, v, params)


@timed("ClaheEqualize")
def clahe_equalize(volume: StructuredVolume, params: ClaheParams) -> None:
    """In-place CLAHE (filters.py:204-245); host-resident volumes are staged
    through HBM."""
    _validate(volume, params)
    with device_resident(volume) as v:
        _clahe_in_hbm(v, params)


def _clahe_in_hbm(volume: StructuredVolume, params: ClaheParams) -> None:
    keep: list = []
    h, a = _histograms(volume, params, keep)
    maps = _mappings_from_hist(h, volume, params)
    dev = volume.data.device
    d, c = volume.dims, params.brick_counts
    lo_w = [_blend_coords(d[ax], _axis_edges(d[ax], c[ax])) for ax in range(3)]
    t_maps = _device(maps.reshape(-1), dev)
    t_lo = _device(np.concatenate([lo_w[0][0], lo_w[1][0], lo_w[2][0]]).astype(np.int32), dev)
    t_w = _device(np.concatenate([lo_w[0][1], lo_w[1][1], lo_w[2][1]]).astype(np.float64), dev)
    keep += [t_maps, t_lo, t_w]
    a.mappings, a.blend_lo, a.blend_w = t_maps.data_ptr(), t_lo.data_ptr(), t_w.data_ptr()
    # the device tables in `keep` are freed in stream order (torch caching
    # allocator), after the blend has read them
    _capi.check(_lib().vkt_clahe_blend(ctypes.byref(a), _stream(dev)))
