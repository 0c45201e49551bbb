"""CPU: host-side API logic (validation, kernels, quantization, error names)."""

import numpy as np
import pytest

import paper_2203_10213_b200 as vk
from conftest import load_filter_cases
from oracle import vkt_oracle as O


class TestKernel:
    def test_even_dims_rejected(self):
        # pkg/tests/test_ops_filter.py:17-19
        with pytest.raises(vk.EvenKernelDims):
            vk.Kernel((2, 3, 3), np.zeros(18))
        with pytest.raises(vk.EvenKernelDims):
            vk.Kernel((3, 0, 3), np.zeros(0))
        with pytest.raises(vk.EvenKernelDims):
            vk.gaussian_kernel(1.0, 4)
        with pytest.raises(vk.EvenKernelDims):
            vk.box_kernel(2)

    def test_error_names_match_reference(self):
        assert vk.EvenKernelDims("x").name == "EvenKernelDims"
        assert vk.InvalidArgument("x").name == "InvalidArgument"
        assert vk.AllocationFailure("x").name == "AllocationFailure"
        assert issubclass(vk.EvenKernelDims, vk.VktError)

    def test_nonfinite_weights_rejected(self):
        w = np.zeros(27)
        w[3] = np.nan
        with pytest.raises(vk.InvalidArgument):
            vk.Kernel((3, 3, 3), w)

    def test_sigma_validation(self):
        with pytest.raises(vk.InvalidArgument):
            vk.gaussian_kernel(0.0)

    def test_gaussian_is_normalized(self):
        k = vk.gaussian_kernel(1.0, 3)
        assert k.weights.sum() == pytest.approx(1.0)
        assert tuple(k.dims) == (3, 3, 3)
        assert tuple(vk.gaussian_kernel(1.0).dims) == (5, 5, 5)
        assert tuple(vk.gaussian_kernel(1.5).dims) == (7, 7, 7)

    def test_weights_bit_identical_to_reference_fixtures(self):
        for c in load_filter_cases():
            n = c["name"]
            if n.startswith("gauss3/"):
                assert np.array_equal(vk.gaussian_kernel(1.0, 3).weights, c["weights"])
            elif n.startswith("gauss5/"):
                assert np.array_equal(vk.gaussian_kernel(1.0).weights, c["weights"])
            elif n.startswith("gauss7/"):
                assert np.array_equal(vk.gaussian_kernel(1.5).weights, c["weights"])
            elif n.startswith("box5/"):
                assert np.array_equal(vk.box_kernel(5).weights, c["weights"])
            elif n.startswith("lap3/"):
                assert np.array_equal(vk.laplacian_kernel().weights, c["weights"])

    def test_x_fastest_layout(self):
        # filters.py:34-36: flat weights are x-fastest -> shape (z, y, x)
        k = vk.Kernel((3, 1, 1), [1.0, 2.0, 3.0])
        assert k.weights.shape == (1, 1, 3)
        assert k.weights[0, 0, 2] == 3.0
        assert tuple(vk.Kernel((3, 1, 5), np.arange(15)).radius) == (1, 0, 2)

    def test_filter_alias(self):
        assert vk.Filter is vk.Kernel


class TestAddressMode:
    def test_values_match_c_abi(self):
        assert [int(m) for m in vk.AddressMode] == [0, 1, 2, 3]
        assert vk.AddressMode.coerce("mirror") is vk.AddressMode.MIRROR
        assert vk.AddressMode.coerce(2) is vk.AddressMode.CLAMP
        with pytest.raises(vk.InvalidArgument):
            vk.AddressMode.coerce("reflect")


class TestQuantize:
    @pytest.mark.parametrize("fmt", [vk.DataFormat.UINT8, vk.DataFormat.UINT16, vk.DataFormat.FLOAT32])
    def test_scalar_rule_matches_oracle(self, fmt):
        rng = np.random.default_rng(5)
        for lo, hi in ((0.0, 1.0), (-1.0, 3.0), (2.5, 2.75)):
            m = vk.VoxelMapping(lo, hi)
            for v in rng.uniform(lo - 1, hi + 1, size=200):
                got = vk.quantize_scalar(v, fmt, m)
                want = O.quantize(np.array([v]), fmt.value, lo, hi)[0]
                assert got == want and got.dtype == want.dtype

    def test_half_rounds_up(self):
        # pkg/tests/test_core.py:140-144: 0.5 -> 128 for u8
        assert int(vk.quantize_scalar(0.5, vk.DataFormat.UINT8, vk.VoxelMapping(0, 1))) == 128
        assert vk.dequantize_scalar(255, vk.DataFormat.UINT8, vk.VoxelMapping(0, 1)) == 1.0

    def test_mapping_validation(self):
        with pytest.raises(vk.InvalidArgument):
            vk.VoxelMapping(1.0, 1.0)
        with pytest.raises(vk.InvalidArgument):
            vk.VoxelMapping(0.0, float("inf"))

    def test_format_codes(self):
        assert [f.value for f in vk.DataFormat] == [1, 2, 3]
        assert vk.DataFormat.parse("u16") is vk.DataFormat.UINT16
        assert vk.DataFormat.from_code(3) is vk.DataFormat.FLOAT32
        with pytest.raises(vk.InvalidArgument):
            vk.DataFormat.from_code(9)


class TestGeometry:
    def test_clip_and_empty(self):
        b = vk.clip_box(vk.box3i((-5, -5, -5), (99, 99, 99)), vk.full_box((4, 4, 4)))
        assert tuple(b.lower) == (0, 0, 0) and tuple(b.upper) == (4, 4, 4)
        assert vk.box3i((2, 2, 2), (2, 2, 2)).is_empty
        with pytest.raises(vk.InvalidArgument):
            vk.box3i((0, 0), (1, 1, 1))


def test_no_cpu_fallback_without_cuda():
    import torch

    if torch.cuda.is_available():
        pytest.skip("CUDA present")
    with pytest.raises(vk.DeviceFailure):
        vk.StructuredVolume((4, 4, 4), vk.DataFormat.UINT8)


def test_product_package_never_imports_oracle():
    import pathlib

    pkg = pathlib.Path(vk.__file__).parent
    for f in pkg.rglob("*.py"):
        src = f.read_text()
        assert "import oracle" not in src and "from oracle" not in src, f


def test_make_args_weight_cache_follows_the_kernel():
    """make_args caches the flat float64 weights on the Kernel; in-place edits
    and reassignment of Kernel.weights must reach the ABI struct."""
    import ctypes

    import numpy as np

    import paper_2203_10213_b200 as vk
    from paper_2203_10213_b200.filters import make_args

    k = vk.gaussian_kernel(1.0, 3)
    a, keep = make_args(1, 2, (4, 5, 6), vk.DataFormat.UINT8, (0.0, 1.0), k, vk.AddressMode.WRAP,
                        halo_lo=7, z_offset=3, global_nz=9, out_z_begin=1, out_z_end=5, flags=2)
    w = np.ctypeslib.as_array(a.weights, shape=(27,))
    assert np.array_equal(w, k.weights.reshape(-1))
    assert (a.src, a.dst, a.halo_lo, a.halo_hi) == (2, 1, 7, None)
    assert (a.dims.x, a.dims.y, a.dims.z, a.kdims.x, a.address_mode) == (4, 5, 6, 3, int(vk.AddressMode.WRAP))
    assert (a.z_offset, a.global_nz, a.out_z_begin, a.out_z_end, a.flags) == (3, 9, 1, 5, 2)
    k.weights[1, 1, 1] = 0.25  # in place: the cached flat array is a view
    a2, _ = make_args(1, 2, (4, 5, 6), vk.DataFormat.UINT8, (0.0, 1.0), k, vk.AddressMode.CLAMP)
    assert np.ctypeslib.as_array(a2.weights, shape=(27,))[13] == 0.25
    k.weights = np.full((3, 3, 3), 1.0 / 27)  # reassigned: repacked
    a3, keep3 = make_args(1, 2, (4, 5, 6), vk.DataFormat.UINT8, (0.0, 1.0), k, vk.AddressMode.CLAMP)
    assert np.allclose(np.ctypeslib.as_array(a3.weights, shape=(27,)), 1.0 / 27)
    assert ctypes.addressof(a3.weights.contents) == keep3.ctypes.data


def test_fill_bits_matches_the_numpy_quantize_rule():
    """fill_bits (plain float64 arithmetic) == stored_bits(quantize_scalar(...))
    (the numpy restatement of volume.py:102-110) on edge and random values."""
    import numpy as np

    from paper_2203_10213_b200.volume import (DataFormat, VoxelMapping, fill_bits, quantize_scalar,
                                              stored_bits)

    rng = np.random.default_rng(3)
    vals = list(rng.normal(0.5, 1.0, 3000)) + [k / 255 for k in range(256)] + \
        [(k + 0.5) / 255 for k in range(255)] + [k / 65535 for k in range(0, 65536, 97)] + \
        [0.0, -0.0, 1.0, 1e300, -1e300, 3.4e38, float("inf"), -float("inf")]
    for fmt in (DataFormat.UINT8, DataFormat.UINT16, DataFormat.FLOAT32):
        for m in (VoxelMapping(0.0, 1.0), VoxelMapping(-1.0, 3.0), VoxelMapping(0.1, 0.7)):
            for v in vals:
                with np.errstate(over="ignore"):
                    want = stored_bits(quantize_scalar(v, fmt, m), fmt)
                assert fill_bits(v, fmt, m) == want, (fmt, m, v)
