"""CLAHE-3D: host tables (CPU) and the device path against the reference's
own outputs (tests/golden/clahe_cases.npz, oracle/make_golden.py) — bit-exact."""

import math

import numpy as np
import pytest
from hypothesis import given, settings
from hypothesis import strategies as st

import paper_2203_10213_b200 as vk
from paper_2203_10213_b200.clahe import _blend_coords, _clip_counts, _axis_edges
from conftest import GOLDEN

FMT = {1: vk.DataFormat.UINT8, 2: vk.DataFormat.UINT16, 3: vk.DataFormat.FLOAT32}


def _cases():
    z = np.load(GOLDEN / "clahe_cases.npz")
    keys = sorted({k.split("/")[0] for k in z.files})
    out = []
    for k in keys:
        s = z[f"{k}/spec"]
        out.append(dict(key=k, input=z[f"{k}/input"], output=z[f"{k}/output"], maps=z[f"{k}/maps"],
                        fmt=int(s[0]), lo=float(s[1]), hi=float(s[2]),
                        bricks=tuple(int(v) for v in s[3:6]), bins=int(s[6]), clip=float(s[7])))
    return out


# ---- CPU: host-side tables (pkg/tests/test_ops_filter.py:72-82) ----

@given(st.lists(st.integers(0, 500), min_size=4, max_size=64), st.integers(1, 200))
@settings(max_examples=100, deadline=None)
def test_clip_mass_conserved(counts, limit):
    hist = np.asarray(counts, dtype=np.int64)
    clipped = _clip_counts(hist, limit)
    assert clipped.sum() == hist.sum() and np.all(clipped >= 0)


def test_clip_leading_bins_take_remainder():
    clipped = _clip_counts(np.array([10, 0, 0, 0], dtype=np.int64), 4)
    assert clipped.tolist() == [6, 2, 1, 1]


def test_axis_tables():
    e = _axis_edges(10, 3)
    assert e.tolist() == [0, 4, 7, 10]
    lo, w = _blend_coords(10, e)
    assert lo.min() >= 0 and lo.max() <= 1 and np.all((w >= 0) & (w <= 1))
    lo1, w1 = _blend_coords(10, _axis_edges(10, 1))
    assert not lo1.any() and not w1.any()


# ---- GPU: bit-exact against the reference ----

@pytest.mark.gpu
@pytest.mark.parametrize("case", _cases(), ids=lambda c: c["key"])
def test_clahe_bit_exact(case):
    v = vk.StructuredVolume.from_numpy(case["input"], FMT[case["fmt"]], mapping=(case["lo"], case["hi"]))
    params = vk.ClaheParams(case["bricks"], case["bins"], case["clip"])
    maps = vk.brick_mappings(v, params)
    assert np.array_equal(maps, case["maps"])
    vk.clahe_equalize(v, params)
    assert np.array_equal(v.to_numpy().view(np.uint8), case["output"].view(np.uint8))


@pytest.mark.gpu
def test_clahe_reference_unit_properties():
    # pkg/tests/test_ops_filter.py:86-135
    v = vk.StructuredVolume((8, 8, 8), vk.DataFormat.UINT8)
    vk.fill(v, 0.3)
    vk.clahe_equalize(v, vk.ClaheParams((2, 2, 2), 64, 4.0))
    a = v.to_numpy()
    assert np.all(a == a[0, 0, 0])
    rng = np.random.default_rng(1234)
    v = vk.StructuredVolume.from_numpy(rng.integers(0, 256, (32, 32, 32), dtype=np.uint8), mapping=(-1.0, 2.0))
    vk.clahe_equalize(v, vk.ClaheParams((2, 2, 2), 256, 4.0))
    m = v.mapped_numpy()
    assert m.min() >= -1.0 and m.max() <= 2.0
    for bricks in ((2, 2, 2), (3, 1, 2), (1, 4, 1)):
        for clip in (1.5, 4.0, math.inf):
            w = vk.StructuredVolume.from_numpy(rng.integers(0, 256, (16, 16, 16), dtype=np.uint8))
            maps = vk.brick_mappings(w, vk.ClaheParams(bricks, 64, clip))
            assert np.all(np.diff(maps, axis=-1) >= 0.0) and np.allclose(maps[..., -1], 1.0)
    with pytest.raises(vk.InvalidArgument):
        vk.clahe_equalize(v, vk.ClaheParams((1, 1, 1), 1, math.inf))
    with pytest.raises(vk.InvalidArgument):
        vk.clahe_equalize(v, vk.ClaheParams((64, 1, 1), 16, math.inf))


@pytest.mark.gpu
def test_clahe_large_u16_runs_and_is_monotone_per_brick():
    import torch

    v = vk.synthetic_device((256, 256, 256), vk.DataFormat.UINT16, seed=2)
    params = vk.ClaheParams((4, 4, 4), 256, 3.0)
    maps = vk.brick_mappings(v, params)
    assert maps.shape == (4, 4, 4, 256) and np.allclose(maps[..., -1], 1.0)
    vk.clahe_equalize(v, params)
    torch.cuda.synchronize()


@pytest.mark.gpu
def test_cli_clahe_matches_library(tmp_path):
    import subprocess
    import sys

    src = GOLDEN / "vol_u16.vkt"
    out = tmp_path / "c.vkt"
    r = subprocess.run([sys.executable, "-m", "paper_2203_10213_b200", "clahe", "--bricks", "2", "2", "2",
                        "--bins", "64", "--clip", "3", "-i", str(src), "-o", str(out)],
                       capture_output=True, timeout=300)
    assert r.returncode == 0, r.stderr
    v = vk.read_volume(src)
    vk.clahe_equalize(v, vk.ClaheParams((2, 2, 2), 64, 3.0))
    assert out.read_bytes() == vk.volume_to_bytes(v)
