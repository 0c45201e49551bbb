"""The separable kernel (csrc/filter_sep.cuh) against the oracle.

Rank-1 weights -- gaussian_kernel (filters.py:45-58), box_kernel
(filters.py:61-66), any outer product fz (x) fy (x) fx -- run as three fused
1-D passes under the "auto" path.  Contract as everywhere:
integer voxels within 1 LSB, f32 within rtol 1e-5 (plus atol 1e-5 for
kernels with negative weights).  f32 outputs whose window holds an Inf / NaN
are recomputed on the device by the direct kernel (bitwise its result there);
every output depends only on its own window, whatever the launch split.
"""

import numpy as np
import pytest

import paper_2203_10213_b200 as vk
from conftest import within_contract
from oracle import vkt_oracle as O

pytestmark = pytest.mark.gpu

FMT = {1: vk.DataFormat.UINT8, 2: vk.DataFormat.UINT16, 3: vk.DataFormat.FLOAT32}
MODES = ("wrap", "mirror", "clamp", "border")


def _stored(rng, fmt, shape):
    if fmt == 3:
        return rng.random(shape, dtype=np.float32)
    return rng.integers(0, np.iinfo(O.DTYPE[fmt]).max + 1, size=shape, dtype=O.DTYPE[fmt])


def _run(stored, fmt, w, mode, path="auto", mapping=(0.0, 1.0)):
    vk.set_execution_policy(vk.ExecutionPolicy(filter_path=path))
    try:
        src = vk.StructuredVolume.from_numpy(stored, FMT[fmt], mapping=mapping)
        dst = vk.StructuredVolume(src.dims, src.format, mapping=mapping)
        kz, ky, kx = w.shape
        kernel = vk.Kernel((kx, ky, kz), w.reshape(-1))
        chosen = vk.filter_path(dst, src, kernel, mode)
        vk.ApplyFilter(dst, src, kernel, mode)
        return dst.to_numpy(), chosen
    finally:
        vk.set_execution_policy(vk.ExecutionPolicy())


def _outer(fz, fy, fx):
    return np.asarray(fz)[:, None, None] * np.asarray(fy)[None, :, None] * np.asarray(fx)[None, None, :]


def test_path_choice():
    src = vk.StructuredVolume((64, 16, 8), vk.DataFormat.UINT16)
    dst = vk.StructuredVolume(src.dims, src.format)
    for k in (3, 5, 7, 9):
        assert vk.filter_path(dst, src, vk.gaussian_kernel(1.0, k)) == "separable"
        assert vk.filter_path(dst, src, vk.box_kernel(k)) == "separable"
    assert vk.filter_path(dst, src, vk.laplacian_kernel()) == "tma"  # not rank-1
    rng = np.random.default_rng(0)
    assert vk.filter_path(dst, src, vk.Kernel((5, 5, 5), rng.random(125))) == "tma"
    f = vk.StructuredVolume((64, 16, 8), vk.DataFormat.FLOAT32)
    fd = vk.StructuredVolume(f.dims, f.format)
    assert vk.filter_path(fd, f, vk.gaussian_kernel(1.0, 3)) == "tma"  # f32 3^3: HBM-bound dense
    assert vk.filter_path(fd, f, vk.gaussian_kernel(1.0, 5)) == "separable"
    vk.set_execution_policy(vk.ExecutionPolicy(filter_path="dense"))
    try:
        assert vk.filter_path(dst, src, vk.gaussian_kernel(1.0, 7)) == "tma"
    finally:
        vk.set_execution_policy(vk.ExecutionPolicy())


@pytest.mark.parametrize("fmt", [1, 2, 3])
@pytest.mark.parametrize("k", [3, 5, 7, 9])
@pytest.mark.parametrize("shape", [(23, 37, 80), (20, 33, 141), (9, 70, 300), (3, 2, 5)],
                         ids=lambda s: "x".join(map(str, s)))
def test_separable_vs_oracle_all_modes(fmt, k, shape):
    """Every format x extent x mode on 16-byte rows (TMA direct), odd rows
    (pitched staging), several tiles per axis, and a volume smaller than the
    halo (every tap address-mapped)."""
    rng = np.random.default_rng(31 * k + fmt + shape[2])
    stored = _stored(rng, fmt, shape)
    w = O.gaussian_weights(1.0 if k < 7 else 1.5, k) if k != 5 else O.box_weights(5)
    want_path = "tma" if fmt == 3 and k == 3 else "separable"
    for mode in MODES:
        want = O.apply_filter(stored, fmt, w, mode, workers=1)
        got, path = _run(stored, fmt, w, mode)
        assert path == want_path
        ok, ndiff, dmax = within_contract(got, want, fmt, w)
        assert ok, (mode, ndiff, dmax)


@pytest.mark.parametrize("fmt", [1, 2])
def test_integer_mapping_epilogue(fmt):
    """A non-unit mapping: the epilogue constant c = lo*(sum_w - 1)/(hi-lo)*max
    (volume.py:102-110) with factors whose sum is not 1."""
    rng = np.random.default_rng(5)
    stored = _stored(rng, fmt, (12, 40, 96))
    w = _outer(rng.random(5), rng.random(5), rng.random(5)) * 0.05
    for mode in MODES:
        want = O.apply_filter(stored, fmt, w, mode, -1.5, 2.0, workers=1)
        got, path = _run(stored, fmt, w, mode, mapping=(-1.5, 2.0))
        assert path == "separable"
        ok, ndiff, dmax = within_contract(got, want, fmt, w)
        assert ok, (mode, ndiff, dmax)


@pytest.mark.parametrize("fmt", [1, 2, 3])
@pytest.mark.parametrize("kd", [(9, 1, 1), (1, 7, 1), (1, 1, 5), (3, 5, 7), (7, 3, 5), (5, 5, 1)],
                         ids=lambda k: "x".join(map(str, k)))
def test_anisotropic_rank1(fmt, kd):
    """(kx, ky, kz) outer products pad their factors to the K^3 cube."""
    rng = np.random.default_rng(sum(kd) * 7 + fmt)
    stored = _stored(rng, fmt, (11, 29, 144))
    kx, ky, kz = kd
    w = _outer(rng.random(kz), rng.random(ky), rng.random(kx))
    w /= w.sum()
    for mode in MODES:
        want = O.apply_filter(stored, fmt, w, mode, workers=1)
        got, path = _run(stored, fmt, w, mode)
        assert path == "separable", (kd, path)
        ok, ndiff, dmax = within_contract(got, want, fmt, w)
        assert ok, (mode, ndiff, dmax)


def test_negative_factors_f32():
    """A derivative-of-Gaussian style kernel (mixed signs): atol applies."""
    rng = np.random.default_rng(9)
    stored = rng.random((16, 40, 128), dtype=np.float32) - np.float32(0.5)
    g = np.exp(-0.5 * (np.arange(-3, 4) / 1.2) ** 2)
    w = _outer(g, g, np.arange(-3, 4) * g) / 50.0
    for mode in MODES:
        want = O.apply_filter(stored, 3, w, mode, workers=1)
        got, path = _run(stored, 3, w, mode)
        assert path == "separable"
        ok, ndiff, dmax = within_contract(got, want, 3, w)
        assert ok, (mode, ndiff, dmax)


@pytest.mark.parametrize("k", [5, 7, 9])
def test_nonfinite_f32_falls_back_to_direct(k):
    """Inf / NaN voxels: the kernel flags them and the direct kernel recomputes
    the outputs it left non-finite -- exactly those whose window holds an Inf
    or NaN -- with the dense arithmetic (0 * Inf = NaN where the reference has
    it).  Every other output keeps its separable value.  All four modes (the
    Wrap / Mirror neighbours of a face voxel included)."""
    rng = np.random.default_rng(k)
    stored = rng.random((14, 30, 130), dtype=np.float32)
    stored[7, 12, 60] = np.inf
    stored[0, 0, 0] = -np.inf
    stored[13, 29, 129] = np.nan
    clean = stored.copy()
    clean[~np.isfinite(clean)] = 0.5
    w = O.gaussian_weights(1.0, k)
    for mode in MODES:
        got, path = _run(stored, 3, w, mode)
        assert path == "separable"
        direct, _ = _run(stored, 3, w, mode, path="direct")
        bad = ~np.isfinite(direct)
        assert bad.any()
        assert np.array_equal(got[bad].view(np.uint32), direct[bad].view(np.uint32)), mode
        sep_clean, _ = _run(clean, 3, w, mode)
        assert np.array_equal(got[~bad].view(np.uint32), sep_clean[~bad].view(np.uint32)), mode
    # the flag is per launch: a finite volume afterwards takes the separable result
    fin = rng.random((14, 30, 130), dtype=np.float32)
    got, _ = _run(fin, 3, w, "clamp")
    ok, ndiff, dmax = within_contract(got, O.apply_filter(fin, 3, w, "clamp", workers=1), 3, w)
    assert ok, (ndiff, dmax)


@pytest.mark.parametrize("mode", MODES)
def test_nonfinite_f32_independent_of_launch_split(mode):
    """The same Inf / NaN volume through the chunked host pipeline (one launch
    per chunk, each with its own flag) and through z-chunked single launches:
    bitwise the whole-volume launch."""
    rng = np.random.default_rng(3)
    stored = rng.random((40, 24, 64), dtype=np.float32)
    stored[3, 5, 7] = np.nan
    stored[21, 10, 30] = np.inf
    w = O.gaussian_weights(1.5, 7)
    kern = vk.Kernel((7, 7, 7), w.reshape(-1))
    want, _ = _run(stored, 3, w, mode)
    for chunk in (2, 9):
        got = vk.apply_filter_host(stored, kern, mode, chunk_planes=chunk)
        assert np.array_equal(got.view(np.uint32), want.view(np.uint32)), chunk


@pytest.mark.parametrize("fmt,k", [(1, 3), (2, 7), (3, 9), (2, 5)])
def test_chunking_invariant(monkeypatch, fmt, k):
    """z chunks restart each CTA's rolling accumulators: any chunk depth gives
    bitwise the same result (each output's sums run in a fixed order)."""
    rng = np.random.default_rng(fmt * 10 + k)
    stored = _stored(rng, fmt, (90, 20, 136))
    w = O.gaussian_weights(1.3, k)
    outs = []
    for zc in (1, 4, 17, 90):
        monkeypatch.setenv("VKT_TMA_ZC", str(zc))
        outs.append(_run(stored, fmt, w, "mirror")[0])
    for o in outs[1:]:
        assert np.array_equal(o.view(np.uint8), outs[0].view(np.uint8))
    ok, ndiff, dmax = within_contract(outs[0], O.apply_filter(stored, fmt, w, "mirror", workers=1), fmt, w)
    assert ok, (ndiff, dmax)


@pytest.mark.parametrize("mode", MODES)
@pytest.mark.parametrize("fmt,k", [(2, 7), (1, 3), (3, 5)])
def test_face_tiles_first_covers_every_tile(monkeypatch, mode, fmt, k):
    """tma::edge_first permutes the blocks (face tiles of the last z chunk, or
    of every chunk under Wrap, first): on a grid of 3 x 4+ tiles and several
    z chunks every tile is still computed exactly once."""
    rng = np.random.default_rng(k + 10 * fmt)
    stored = _stored(rng, fmt, (70, 50, 300))
    w = O.gaussian_weights(1.0, k) if k != 5 else O.box_weights(5)
    monkeypatch.setenv("VKT_TMA_ZC", "16")
    got, path = _run(stored, fmt, w, mode)
    assert path == "separable" or (fmt == 3 and k == 3)
    ok, ndiff, dmax = within_contract(got, O.apply_filter(stored, fmt, w, mode, workers=1), fmt, w)
    assert ok, (ndiff, dmax)


@pytest.mark.parametrize("fmt", [1, 2, 3])
@pytest.mark.parametrize("k", [11, 13, 15, 17, 21])
def test_large_extents(fmt, k):
    """gaussian_kernel's default extent reaches 11 at sigma 2.5, 13 at 3, 15 at
    3.5, 17 at 4 and 21 at 5: those run on the separable kernel too (halos of
    2-3 quads per side), every mode, against the oracle; 23 and up take the
    direct kernel."""
    rng = np.random.default_rng(k * 3 + fmt)
    stored = _stored(rng, fmt, (24, 21, 144))
    sigma = {11: 2.5, 13: 3.0, 15: 3.5, 17: 4.0, 21: 5.0}[k]
    w = O.gaussian_weights(sigma)
    assert w.shape == (k, k, k)
    for mode in MODES:
        want = O.apply_filter(stored, fmt, w, mode, workers=1)
        got, path = _run(stored, fmt, w, mode)
        assert path == "separable"
        ok, ndiff, dmax = within_contract(got, want, fmt, w)
        assert ok, (mode, ndiff, dmax)
    src = vk.StructuredVolume((64, 16, 8), vk.DataFormat.UINT16)
    dst = vk.StructuredVolume(src.dims, src.format)
    assert vk.filter_path(dst, src, vk.gaussian_kernel(5.5)) == "direct"  # 23^3


@pytest.mark.parametrize("fmt", [1, 3])
def test_large_extent_on_a_tiny_volume(fmt):
    """21^3 on a 5 x 2 x 3 volume: every tap address-mapped, most of the
    TMA box outside the volume (the repair table covers it)."""
    rng = np.random.default_rng(21 + fmt)
    stored = _stored(rng, fmt, (3, 2, 5))
    w = O.gaussian_weights(5.0)
    for mode in MODES:
        want = O.apply_filter(stored, fmt, w, mode, workers=1)
        got, path = _run(stored, fmt, w, mode)
        assert path == "separable"
        ok, ndiff, dmax = within_contract(got, want, fmt, w)
        assert ok, (mode, ndiff, dmax)
