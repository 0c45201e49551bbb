"""GPU: the tiled kernel's edge handling on awkward shapes, against the oracle.

Extents smaller than the radius (multi-fold Mirror / Wrap), single cells,
tiles straddling the 128 x 16 tile grid, and rows that are not 16-byte
multiples (pitched staging) — for every address mode, kernel extent and
voxel format.  The fast path must stay within the contract and the EXACT
path bit-exact.
"""

import numpy as np
import pytest

import paper_2203_10213_b200 as vk
from conftest import within_contract
from oracle import vkt_oracle as O

pytestmark = pytest.mark.gpu

FMT = {1: vk.DataFormat.UINT8, 2: vk.DataFormat.UINT16, 3: vk.DataFormat.FLOAT32}
SHAPES = [(1, 1, 1), (2, 3, 4), (3, 5, 2), (5, 4, 7), (17, 3, 9), (16, 16, 3), (129, 17, 5),
          (130, 33, 3), (64, 2, 6), (144, 20, 4)]


def _run(stored, fmt, w, mode, path):
    vk.set_execution_policy(vk.ExecutionPolicy(filter_path=path))
    try:
        src = vk.StructuredVolume.from_numpy(stored, FMT[fmt])
        dst = vk.StructuredVolume(src.dims, src.format)
        k = w.shape[0]
        vk.ApplyFilter(dst, src, vk.Kernel((k, k, k), w.reshape(-1)), mode)
        return dst.to_numpy()
    finally:
        vk.set_execution_policy(vk.ExecutionPolicy())


@pytest.mark.parametrize("shape", SHAPES, ids=lambda s: "x".join(map(str, s)))
@pytest.mark.parametrize("fmt", [1, 2, 3])
def test_awkward_shapes_all_modes_and_extents(shape, fmt):
    rng = np.random.default_rng(hash((shape, fmt)) % 2**32)
    nx, ny, nz = shape
    stored = (rng.random((nz, ny, nx), dtype=np.float32) if fmt == 3 else
              rng.integers(0, np.iinfo(O.DTYPE[fmt]).max + 1, size=(nz, ny, nx), dtype=O.DTYPE[fmt]))
    for k in (3, 5, 7):
        w = rng.random((k, k, k))
        w /= w.sum()
        for mode in ("wrap", "mirror", "clamp", "border"):
            want = O.apply_filter(stored, fmt, w, mode, workers=1)
            got = _run(stored, fmt, w, mode, "auto")
            ok, ndiff, dmax = within_contract(got, want, fmt, w)
            assert ok, (shape, k, mode, ndiff, dmax)
            exact = _run(stored, fmt, w, mode, "exact")
            assert np.array_equal(exact.view(np.uint8), want.view(np.uint8)), (shape, k, mode)


@pytest.mark.parametrize("fmt", [1, 2, 3])
@pytest.mark.parametrize("k", [3, 5, 7])
def test_interior_tiles_at_z_boundaries(fmt, k):
    """Tiles with no x/y edge still meet the z boundary (zero planes under
    Border, mapped planes otherwise): 3 x 3 tiles, the middle one interior."""
    rng = np.random.default_rng(1000 * fmt + k)
    nx, ny, nz = 384, 48, 5
    stored = (rng.random((nz, ny, nx), dtype=np.float32) if fmt == 3 else
              rng.integers(0, np.iinfo(O.DTYPE[fmt]).max + 1, size=(nz, ny, nx), dtype=O.DTYPE[fmt]))
    w = rng.random((k, k, k))
    w /= w.sum()
    for mode in ("wrap", "mirror", "clamp", "border"):
        want = O.apply_filter(stored, fmt, w, mode, workers=1)
        got = _run(stored, fmt, w, mode, "auto")
        ok, ndiff, dmax = within_contract(got, want, fmt, w)
        assert ok, (k, mode, ndiff, dmax)


@pytest.mark.parametrize("fmt", [1, 2, 3])
@pytest.mark.parametrize("shape", [(140, 40, 11), (33, 7, 5), (256, 20, 3)], ids=lambda s: "x".join(map(str, s)))
def test_tiled_k9_all_modes(shape, fmt):
    """9x9x9 runs on the tiled kernel (R = 4, the largest halo its layout
    takes): within contract against the oracle under every address mode."""
    rng = np.random.default_rng(900 + fmt)
    nx, ny, nz = shape
    stored = (rng.random((nz, ny, nx), dtype=np.float32) if fmt == 3 else
              rng.integers(0, np.iinfo(O.DTYPE[fmt]).max + 1, size=(nz, ny, nx), dtype=O.DTYPE[fmt]))
    w = rng.random((9, 9, 9))
    w /= w.sum()
    src = vk.StructuredVolume.from_numpy(stored, FMT[fmt])
    dst = vk.StructuredVolume(src.dims, src.format)
    assert vk.filter_path(dst, src, vk.Kernel((9, 9, 9), w.reshape(-1))) == "tma"
    for mode in ("wrap", "mirror", "clamp", "border"):
        want = O.apply_filter(stored, fmt, w, mode, workers=1)
        got = _run(stored, fmt, w, mode, "auto")
        ok, ndiff, dmax = within_contract(got, want, fmt, w)
        assert ok, (shape, mode, ndiff, dmax)


@pytest.mark.parametrize("fmt", [1, 2])
@pytest.mark.parametrize("kd", [(3, 1, 5), (5, 5, 1), (1, 3, 3), (7, 3, 1), (9, 1, 1), (3, 3, 5)],
                         ids=lambda k: "x".join(map(str, k)))
def test_anisotropic_integer_kernels_on_the_tiled_path(kd, fmt):
    """Anisotropic integer kernels run on the tiled kernel, embedded in a K^3
    cube of zero weights: bit-identical to the direct kernel (same FP32 tap
    sequence; the zero taps add exact +0) and within contract of the oracle."""
    rng = np.random.default_rng(77 + fmt)
    stored = rng.integers(0, np.iinfo(O.DTYPE[fmt]).max + 1, size=(7, 21, 140), dtype=O.DTYPE[fmt])
    w = rng.random(kd[::-1])
    w /= w.sum()
    src = vk.StructuredVolume.from_numpy(stored, FMT[fmt])
    dst = vk.StructuredVolume(src.dims, src.format)
    kernel = vk.Kernel(kd, w.reshape(-1))
    # a 1-D kernel is rank-1 and takes the separable kernel under "auto"
    auto = "separable" if sum(d > 1 for d in kd) == 1 else "tma"
    assert vk.filter_path(dst, src, kernel) == auto
    vk.set_execution_policy(vk.ExecutionPolicy(filter_path="dense"))
    try:
        assert vk.filter_path(dst, src, kernel) == "tma"
    finally:
        vk.set_execution_policy(vk.ExecutionPolicy())

    def run(mode, path):
        vk.set_execution_policy(vk.ExecutionPolicy(filter_path=path))
        try:
            vk.ApplyFilter(dst, src, kernel, mode)
            return dst.to_numpy()
        finally:
            vk.set_execution_policy(vk.ExecutionPolicy())

    for mode in ("wrap", "mirror", "clamp", "border"):
        want = O.apply_filter(stored, fmt, w, mode, workers=1)
        for path in ("auto", "dense"):
            got = run(mode, path)
            ok, ndiff, dmax = within_contract(got, want, fmt, w)
            assert ok, (kd, mode, path, ndiff, dmax)
        assert np.array_equal(got, run(mode, "direct")), (kd, mode)


@pytest.mark.parametrize("kd", [(5, 5, 1), (7, 7, 3), (9, 9, 1), (5, 5, 3)], ids=lambda k: "x".join(map(str, k)))
def test_anisotropic_f32_z_padded_on_the_tiled_path(kd):
    """f32 kernels with kx = ky > kz run on the tiled kernel padded in z, the
    padding planes skipped outright: bit-identical to the direct kernel, Inf /
    NaN voxels included (a zero-weight tap would have turned Inf into NaN)."""
    rng = np.random.default_rng(5 + kd[2])
    stored = rng.random((9, 23, 140), dtype=np.float32)
    stored[4, 10, 70] = np.inf
    stored[2, 5, 3] = np.nan
    w = rng.random(kd[::-1])
    w /= w.sum()
    src = vk.StructuredVolume.from_numpy(stored, vk.DataFormat.FLOAT32)
    dst = vk.StructuredVolume(src.dims, src.format)
    kernel = vk.Kernel(kd, w.reshape(-1))
    assert vk.filter_path(dst, src, kernel) == "tma"

    def run(mode, path):
        vk.set_execution_policy(vk.ExecutionPolicy(filter_path=path))
        try:
            vk.ApplyFilter(dst, src, kernel, mode)
            return dst.to_numpy()
        finally:
            vk.set_execution_policy(vk.ExecutionPolicy())

    finite = stored.copy()
    finite[~np.isfinite(finite)] = 0.5
    for mode in ("wrap", "mirror", "clamp", "border"):
        got = run(mode, "auto")
        assert np.array_equal(got.view(np.uint32), run(mode, "direct").view(np.uint32)), (kd, mode)
    src2 = vk.StructuredVolume.from_numpy(finite, vk.DataFormat.FLOAT32)
    vk.ApplyFilter(dst, src2, kernel, "clamp")
    ok, ndiff, dmax = within_contract(dst.to_numpy(), O.apply_filter(finite, 3, w, "clamp", workers=1), 3, w)
    assert ok, (kd, ndiff, dmax)


@pytest.mark.parametrize("kd", [(3, 1, 5), (5, 3, 5), (3, 3, 1), (1, 3, 3), (7, 5, 3), (9, 1, 1),
                                (1, 1, 9), (1, 7, 1)],
                         ids=lambda k: "x".join(map(str, k)))
@pytest.mark.parametrize("nx", [140, 141])
def test_anisotropic_f32_cube(kd, nx):
    """Anisotropic f32 kernels on the tiled kernels.  K >= 5 cubes run only
    the real taps (x extent templated, padding rows / planes skipped), so they
    match the direct kernel bitwise on any volume, Inf / NaN included; K = 3
    cubes run behind an on-device Inf/NaN scan (finite: tiled, exact +0 zero
    taps; otherwise the direct kernel).  1-D kernels are rank-1 and take the
    separable kernel under "auto"."""
    rng = np.random.default_rng(11 + sum(kd) + nx)
    finite = rng.random((9, 23, nx), dtype=np.float32) - np.float32(0.25)
    w = rng.random(kd[::-1]) - 0.2
    kernel = vk.Kernel(kd, w.reshape(-1))
    dst = vk.StructuredVolume((nx, 23, 9), vk.DataFormat.FLOAT32)

    def run(stored, mode, path):
        src = vk.StructuredVolume.from_numpy(stored, vk.DataFormat.FLOAT32)
        vk.set_execution_policy(vk.ExecutionPolicy(filter_path=path))
        try:
            vk.ApplyFilter(dst, src, kernel, mode)
            return dst.to_numpy()
        finally:
            vk.set_execution_policy(vk.ExecutionPolicy())

    src = vk.StructuredVolume.from_numpy(finite, vk.DataFormat.FLOAT32)
    # 1-D kernels with K >= 5 are rank-1: the separable kernel under "auto"
    # (within contract; Inf / NaN inputs fall back to the direct kernel)
    sep = sum(d > 1 for d in kd) == 1 and max(kd) >= 5
    assert vk.filter_path(dst, src, kernel) == ("separable" if sep else "tma")
    bad = finite.copy()
    bad[4, 10, 70] = np.inf
    bad[2, 5, 3] = np.nan
    for mode in ("wrap", "mirror", "clamp", "border"):
        want = O.apply_filter(finite, 3, w, mode, workers=1)
        got = run(finite, mode, "dense")
        assert np.array_equal(got, run(finite, mode, "direct")), (kd, mode)
        ok, ndiff, dmax = within_contract(got, want, 3, w)
        assert ok, (kd, mode, ndiff, dmax)
        ok, ndiff, dmax = within_contract(run(finite, mode, "auto"), want, 3, w)
        assert ok, (kd, mode, "auto", ndiff, dmax)
        direct_bad = run(bad, mode, "direct")
        assert np.array_equal(run(bad, mode, "dense").view(np.uint32), direct_bad.view(np.uint32)), (kd, mode)
        # auto: the separable kernel recomputes exactly the non-finite outputs
        # with the dense arithmetic (bitwise the direct kernel there); the rest
        # keep their separable values, within contract
        got = run(bad, mode, "auto")
        nf = ~np.isfinite(direct_bad)
        assert np.array_equal(got[nf].view(np.uint32), direct_bad[nf].view(np.uint32)), (kd, mode)
        if sep:
            ok, ndiff, dmax = within_contract(got[~nf], direct_bad[~nf], 3, w)
            assert ok, (kd, mode, "auto finite", ndiff, dmax)
        else:
            assert np.array_equal(got.view(np.uint32), direct_bad.view(np.uint32)), (kd, mode)


@pytest.mark.parametrize("zc", [171, 200, 397])
@pytest.mark.parametrize("fmt,k", [(2, 7), (3, 7), (2, 9), (3, 9), (1, 5), (3, 3)])
def test_deep_z_chunks_match_direct(monkeypatch, zc, fmt, k):
    """K >= 7 on big volumes runs ~171-plane z chunks (filter_tma.cu); forced
    deep chunks (VKT_TMA_ZC, the diagnostics override) on a volume small
    enough for the direct kernel stay bit-identical to it."""
    rng = np.random.default_rng(zc + 10 * k + fmt)
    shape = (400, 20, 136)
    stored = (rng.random(shape, dtype=np.float32) if fmt == 3 else
              rng.integers(0, 256 if fmt == 1 else 65536, size=shape).astype(np.uint8 if fmt == 1 else np.uint16))
    w = rng.random((k, k, k))
    w /= w.sum()
    monkeypatch.setenv("VKT_TMA_ZC", str(zc))
    for mode in ("wrap", "clamp"):
        got = _run(stored, fmt, w, mode, "auto")
        assert np.array_equal(got.view(np.uint8), _run(stored, fmt, w, mode, "direct").view(np.uint8)), mode
