"""GPU parity: the CUDA path vs the reference fixtures and the oracle.

Contract: Fill/FillRange bit-exact; integer voxels within
1 LSB; f32 within |d| <= 1e-5*|ref| + 1e-5.  The EXACT_F64 path must be
bit-identical to the reference.  Every kernel path (tiled TMA, direct) must
agree bit-for-bit with each other, so a path switch never changes results.
Rank-1 kernels (gaussian_kernel, box_kernel) take the separable kernel under
"auto" -- within contract, not bitwise; "dense" runs them on the dense tiled
kernels, which stay bit-identical to the direct kernel.
"""

import numpy as np
import pytest

import paper_2203_10213_b200 as vk
from conftest import load_fill_cases, load_filter_cases, within_contract, GOLDEN
from oracle import vkt_oracle as O

pytestmark = pytest.mark.gpu

CASES = load_filter_cases()
FMT = {1: vk.DataFormat.UINT8, 2: vk.DataFormat.UINT16, 3: vk.DataFormat.FLOAT32}


def run_filter(stored, fmt, weights, mode, lo=0.0, hi=1.0, path="auto"):
    import torch

    src = vk.StructuredVolume.from_numpy(stored, FMT[fmt], mapping=(lo, hi))
    dst = vk.StructuredVolume(src.dims, src.format, mapping=(lo, hi))
    kz, ky, kx = weights.shape
    k = vk.Kernel((kx, ky, kz), weights.reshape(-1))
    vk.set_execution_policy(vk.ExecutionPolicy(filter_path=path))
    try:
        vk.ApplyFilter(dst, src, k, vk.AddressMode.coerce(mode))
        torch.cuda.synchronize()
    finally:
        vk.set_execution_policy(vk.ExecutionPolicy())
    # snapshot semantics: the source is untouched
    assert np.array_equal(src.to_numpy(), stored)
    return dst.to_numpy()


@pytest.mark.parametrize("case", CASES, ids=[c["name"] for c in CASES])
def test_fast_path_within_contract(case):
    got = run_filter(case["input"], case["fmt"], case["weights"], case["mode"], case["lo"], case["hi"])
    ok, ndiff, dmax = within_contract(got, case["output"], case["fmt"], case["weights"])
    assert ok, f"{case['name']}: {ndiff} cells differ, max {dmax}"


@pytest.mark.parametrize("case", CASES, ids=[c["name"] for c in CASES])
def test_exact_path_bit_identical(case):
    got = run_filter(case["input"], case["fmt"], case["weights"], case["mode"], case["lo"],
                     case["hi"], path="exact")
    assert np.array_equal(got.view(np.uint8), case["output"].view(np.uint8)), case["name"]


@pytest.mark.parametrize("case", CASES[::7], ids=[c["name"] for c in CASES[::7]])
def test_direct_and_dense_paths_bit_identical(case):
    a = run_filter(case["input"], case["fmt"], case["weights"], case["mode"], case["lo"], case["hi"],
                   path="dense")
    b = run_filter(case["input"], case["fmt"], case["weights"], case["mode"], case["lo"], case["hi"],
                   path="direct")
    assert np.array_equal(a.view(np.uint8), b.view(np.uint8))


@pytest.mark.parametrize("fmt", [1, 2, 3])
@pytest.mark.parametrize("mode", ["clamp", "wrap", "mirror", "border"])
@pytest.mark.parametrize("k", [3, 5, 7])
def test_tiled_shapes_vs_oracle(fmt, mode, k):
    """Shapes the tiled kernel takes (16-byte rows), several tiles per axis."""
    rng = np.random.default_rng(1000 * fmt + k)
    dims = (80, 37, 23)  # x multiple of 16 -> TMA-eligible for every format
    stored = (rng.random((dims[2], dims[1], dims[0]), dtype=np.float32) if fmt == 3 else
              rng.integers(0, np.iinfo(O.DTYPE[fmt]).max + 1, size=dims[::-1], dtype=O.DTYPE[fmt]))
    w = O.gaussian_weights(1.0, k) if k != 5 else O.box_weights(5)
    want = O.apply_filter(stored, fmt, w, mode)
    got = run_filter(stored, fmt, w, mode)
    ok, ndiff, dmax = within_contract(got, want, fmt, w)
    assert ok, (ndiff, dmax)
    dense = run_filter(stored, fmt, w, mode, path="dense")
    direct = run_filter(stored, fmt, w, mode, path="direct")
    assert np.array_equal(dense.view(np.uint8), direct.view(np.uint8))


def test_bench_fixture_u8_gauss3():
    z = np.load(GOLDEN / "bench_case.npz")
    got = run_filter(z["input"], 1, O.gaussian_weights(1.0, 3), "clamp")
    ok, ndiff, dmax = within_contract(got, z["output"], 1, O.gaussian_weights(1.0, 3))
    assert ok, (ndiff, dmax)


# ---- the reference's own ApplyFilter unit tests (pkg/tests/test_ops_filter.py) ----

def test_delta_kernel_fixed_point():
    rng = np.random.default_rng(1234)
    for fmt in (1, 2, 3):
        v = vk.synthetic_structured((6, 6, 6), FMT[fmt], seed=5)
        before = v.data.to_bytes()
        w = np.zeros((3, 3, 3))
        w[1, 1, 1] = 1.0
        vk.apply_filter(v, vk.Kernel((3, 3, 3), w))
        assert v.data.to_bytes() == before
    del rng


def test_box_kernel_on_constant():
    v = vk.StructuredVolume((5, 5, 5), vk.DataFormat.FLOAT32)
    vk.fill(v, 0.625)
    vk.apply_filter(v, vk.Kernel((3, 3, 3), np.full((3, 3, 3), 1 / 27)))
    assert np.allclose(v.to_numpy(), 0.625, atol=1e-7)


def test_gaussian_matches_triple_loop_oracle():
    rng = np.random.default_rng(1234)
    stored = rng.random((8, 8, 8), dtype=np.float32)
    v = vk.StructuredVolume.from_numpy(stored)
    k = vk.gaussian_kernel(1.0, 3)
    vk.apply_filter(v, k)
    expected = O.convolve_scalar(stored.astype(np.float64), k.weights)
    assert np.max(np.abs(v.mapped_numpy() - expected)) < 1e-5


def test_asymmetric_kernel_orientation():
    v = vk.StructuredVolume((4, 1, 1), vk.DataFormat.FLOAT32)
    v.upload(np.array([1.0, 2.0, 3.0, 4.0], dtype=np.float32))
    w = np.zeros((1, 1, 3))
    w[0, 0, 2] = 1.0
    vk.apply_filter(v, vk.Kernel((3, 1, 1), w))
    assert v.to_numpy()[0, 0, :].tolist() == [2.0, 3.0, 4.0, 4.0]


def test_asymmetric_orientation_all_axes_and_modes():
    vals = np.arange(1, 6, dtype=np.float32)
    want = {"clamp": [2, 3, 4, 5, 5], "wrap": [2, 3, 4, 5, 1],
            "mirror": [2, 3, 4, 5, 5], "border": [2, 3, 4, 5, 0]}
    for axis in range(3):
        dims = [1, 1, 1]
        dims[axis] = 5
        kd = [1, 1, 1]
        kd[axis] = 3
        w = np.zeros(3)
        w[2] = 1.0
        for mode, exp in want.items():
            v = vk.StructuredVolume(tuple(dims), vk.DataFormat.FLOAT32)
            v.upload(vals)
            vk.apply_filter(v, vk.Kernel(tuple(kd), w), mode)
            assert v.to_numpy().reshape(-1).tolist() == exp, (axis, mode)


def test_nonnegative_normalized_kernel_preserves_range():
    rng = np.random.default_rng(1234)
    stored = rng.random((8, 8, 8), dtype=np.float32)
    v = vk.StructuredVolume.from_numpy(stored)
    lo, hi = float(stored.min()), float(stored.max())
    vk.apply_filter(v, vk.gaussian_kernel(0.8, 5))
    out = v.to_numpy()
    assert out.min() >= lo - 1e-6 and out.max() <= hi + 1e-6


def test_even_kernel_rejected_before_launch():
    with pytest.raises(vk.EvenKernelDims):
        vk.Kernel((2, 3, 3), np.zeros(18))


def test_dims_mismatch():
    a = vk.StructuredVolume((4, 4, 4), vk.DataFormat.UINT8)
    b = vk.StructuredVolume((4, 4, 5), vk.DataFormat.UINT8)
    with pytest.raises(vk.DimsMismatch):
        vk.ApplyFilter(a, b, vk.gaussian_kernel(1.0, 3))


# ---- Fill / FillRange: bit-exact (pkg/tests/test_ops_core.py:11-48) ----

@pytest.mark.parametrize("case", load_fill_cases(), ids=lambda c: c["key"])
def test_fill_range_bit_exact(case):
    import torch

    v = vk.StructuredVolume.from_numpy(case["input"], FMT[case["fmt"]], mapping=(case["lo"], case["hi"]))
    vk.fill_range(v, vk.box3i(case["lower"], case["upper"]), case["value"])
    torch.cuda.synchronize()
    assert v.data.to_bytes() == case["output"].tobytes()


def test_fill_session_fidelity():
    v = vk.create_structured_volume((64, 64, 64), vk.DataFormat.UINT8, (1, 1, 1), (0, 1))
    vk.FillRange(v, vk.box3i((1, 1, 1), (63, 63, 63)), 1.0)
    m = v.mapped_numpy()
    assert int((m == 1.0).sum()) == 238_328
    assert int((m == 0.0).sum()) == 23_816


def test_fill_half_quantizes():
    v = vk.StructuredVolume((8, 8, 8), vk.DataFormat.UINT8)
    vk.Fill(v, 0.5)
    assert np.all(v.to_numpy() == 128)
    assert v.get_value((3, 3, 3)) == pytest.approx(128 / 255)


def test_fill_unaligned_boxes_all_formats():
    rng = np.random.default_rng(3)
    for fmt in (1, 2, 3):
        for _ in range(12):
            dims = tuple(int(d) for d in rng.integers(1, 70, size=3))
            lo = tuple(int(v) for v in rng.integers(-3, 40, size=3))
            hi = tuple(int(v) for v in rng.integers(0, 80, size=3))
            base = (rng.random(dims[::-1], dtype=np.float32) if fmt == 3 else
                    rng.integers(0, 200, size=dims[::-1]).astype(O.DTYPE[fmt]))
            v = vk.StructuredVolume.from_numpy(base, FMT[fmt])
            vk.fill_range(v, (lo, hi), 0.3)
            want = O.fill_range(base, fmt, lo, hi, 0.3)
            assert v.data.to_bytes() == want.tobytes()


def test_fill_boxes_on_16_byte_rows_all_formats():
    """Rows that are 16-byte multiples take the flattened short-segment fill
    (fill_segs_kernel): every head / vector / tail split of the box rows."""
    rng = np.random.default_rng(5)
    for fmt, nx in ((1, 64), (2, 40), (3, 20)):
        dims = (nx, 13, 6)
        for lx in range(0, 17):
            for w in (1, 3, 5, 16, 17, 23, nx - lx):
                hx = min(nx, lx + w)
                if hx <= lx or (lx == 0 and hx == nx):
                    continue
                lo, hi = (lx, 2, 1), (hx, 11, 5)
                base = (rng.random(dims[::-1], dtype=np.float32) if fmt == 3 else
                        rng.integers(0, 200, size=dims[::-1]).astype(O.DTYPE[fmt]))
                v = vk.StructuredVolume.from_numpy(base, FMT[fmt])
                vk.fill_range(v, (lo, hi), 0.7)
                want = O.fill_range(base, fmt, lo, hi, 0.7)
                assert v.data.to_bytes() == want.tobytes(), (fmt, lo, hi)
