"""CPU: pin the oracle against the reference's own outputs (tests/golden)."""

import math

import numpy as np
import pytest
from hypothesis import given, settings
from hypothesis import strategies as st

from conftest import load_fill_cases, load_filter_cases, GOLDEN
from oracle import vkt_oracle as O

CASES = load_filter_cases()


@pytest.mark.parametrize("case", CASES, ids=[c["name"] for c in CASES])
def test_oracle_bit_identical_to_reference(case):
    got = O.apply_filter(case["input"], case["fmt"], case["weights"], case["mode"],
                         case["lo"], case["hi"], workers=1)
    assert got.dtype == case["output"].dtype
    assert np.array_equal(got.view(np.uint8), case["output"].view(np.uint8)), case["name"]


def test_oracle_threads_and_z_chunks_bit_identical():
    c = next(c for c in CASES if c["name"].startswith("gauss7/u16") and c["input"].shape[0] >= 7)
    full = O.apply_filter(c["input"], c["fmt"], c["weights"], c["mode"], c["lo"], c["hi"], workers=4)
    nz = c["input"].shape[0]
    parts = [O.apply_filter(c["input"], c["fmt"], c["weights"], c["mode"], c["lo"], c["hi"],
                            z_range=(a, b), workers=1)
             for a, b in ((0, 2), (2, 5), (5, nz))]
    assert np.array_equal(np.concatenate(parts), full)
    assert np.array_equal(full, c["output"])


def test_pad_closed_forms_match_numpy():
    for n in range(1, 7):
        for r in range(0, 8):
            base = np.arange(n)
            for mode, npmode in (("wrap", "wrap"), ("mirror", "symmetric"), ("clamp", "edge")):
                want = np.pad(base, r, mode=npmode)
                got = [O.map_index(i, n, mode) for i in range(-r, n + r)]
                assert list(want) == got, (n, r, mode)


def test_scalar_loop_oracle_agrees_on_small_cases():
    for c in CASES[:40]:
        if c["input"].size > 400:
            continue
        mapped = O.dequantize(c["input"], c["fmt"], c["lo"], c["hi"])
        border = O.dequantize(np.zeros(1, O.DTYPE[c["fmt"]]), c["fmt"], c["lo"], c["hi"])[0]
        acc = O.convolve_scalar(mapped, c["weights"], c["mode"], border)
        got = O.quantize(acc, c["fmt"], c["lo"], c["hi"])
        if c["fmt"] == 3:
            assert np.max(np.abs(got.astype(np.float64) - c["output"])) <= 1e-6
        else:
            assert np.max(np.abs(got.astype(np.int64) - c["output"].astype(np.int64))) <= 1


def test_bench_fixture():
    z = np.load(GOLDEN / "bench_case.npz")
    got = O.apply_filter(z["input"], 1, O.gaussian_weights(1.0, 3), "clamp")
    assert np.array_equal(got, z["output"])


@pytest.mark.parametrize("case", load_fill_cases(), ids=lambda c: c["key"])
def test_fill_oracle_bit_identical(case):
    got = O.fill_range(case["input"], case["fmt"], case["lower"], case["upper"], case["value"],
                       case["lo"], case["hi"])
    assert np.array_equal(got.view(np.uint8), case["output"].view(np.uint8))


def test_fig4_session_counts():
    # pkg/tests/test_ops_core.py:12-19 and test_acceptance.py:94-100
    c = load_fill_cases()[0]
    assert int((c["output"] == 255).sum()) == 62**3 == 238_328
    assert int((c["output"] == 0).sum()) == 64**3 - 62**3 == 23_816


@given(stored=st.integers(0, 255), lo=st.floats(-10, 5), width=st.floats(0.25, 20))
@settings(max_examples=60, deadline=None)
def test_quantization_fixed_point_u8(stored, lo, width):
    # pkg/tests/test_core.py:157-163
    hi = lo + width
    m = O.dequantize(np.array([stored], dtype=np.uint8), 1, lo, hi)
    assert int(O.quantize(m, 1, lo, hi)[0]) == stored


def test_gaussian_weights_match_reference_fixture():
    for c in CASES:
        n = c["name"]
        if n.startswith("gauss3/"):
            assert np.array_equal(O.gaussian_weights(1.0, 3), c["weights"])
        if n.startswith("gauss5/"):
            assert np.array_equal(O.gaussian_weights(1.0), c["weights"])
        if n.startswith("gauss7/"):
            assert np.array_equal(O.gaussian_weights(1.5), c["weights"])
        if n.startswith("box5/"):
            assert np.array_equal(O.box_weights(5), c["weights"])
        if n.startswith("lap3/"):
            assert np.array_equal(O.laplacian_weights(), c["weights"])
    assert math.isclose(O.gaussian_weights(1.0, 3).sum(), 1.0)
