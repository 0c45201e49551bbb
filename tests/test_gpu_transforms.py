"""GPU: Flip and Resample bit-exact against the reference (tests/golden/transform_cases.npz)."""

import numpy as np
import pytest

import paper_2203_10213_b200 as vk
from conftest import GOLDEN

pytestmark = pytest.mark.gpu
FMT = {1: vk.DataFormat.UINT8, 2: vk.DataFormat.UINT16, 3: vk.DataFormat.FLOAT32}


def _cases():
    z = np.load(GOLDEN / "transform_cases.npz")
    keys = sorted({k.split("/")[0] for k in z.files})
    return [dict(key=k, **{n: z[f"{k}/{n}"] for n in ("input", "output", "spec", "cell", "flip0", "flip1", "flip2")})
            for k in keys]


@pytest.mark.parametrize("case", _cases(), ids=lambda c: c["key"])
def test_resample_and_flip_bit_exact(case):
    s = case["spec"]
    fmt, lo, hi = int(s[0]), float(s[1]), float(s[2])
    ddims = tuple(int(v) for v in s[3:6])
    dfmt, dlo, dhi = int(s[6]), float(s[7]), float(s[8])
    v = vk.StructuredVolume.from_numpy(case["input"], FMT[fmt], cell_size=(1, 0.5, 2), mapping=(lo, hi))
    r = vk.resample(v, ddims, FMT[dfmt], (dlo, dhi))
    assert np.array_equal(r.to_numpy().view(np.uint8), case["output"].view(np.uint8))
    assert np.allclose(tuple(r.cell_size), case["cell"], rtol=0, atol=0)
    for ax in range(3):
        f = vk.StructuredVolume.from_numpy(case["input"], FMT[fmt], mapping=(lo, hi))
        vk.flip(f, "xyz"[ax])
        assert np.array_equal(f.to_numpy(), case[f"flip{ax}"])


def test_flip_twice_is_identity_large():
    import torch

    v = vk.synthetic_device((512, 256, 128), vk.DataFormat.UINT16, seed=4)
    before = v.data.array.clone()
    for ax in ("x", "y", "z"):
        vk.flip(v, ax)
        vk.flip(v, ax)
    assert torch.equal(v.data.array, before)
    with pytest.raises(vk.InvalidArgument):
        vk.flip(v, "w")


def test_cli_flip_resample_pipe(tmp_path):
    import subprocess
    import sys

    from conftest import GOLDEN as G

    src = G / "vol_u16.vkt"
    cli = [sys.executable, "-m", "paper_2203_10213_b200"]
    first = subprocess.run(cli + ["resample", "--dims", "8", "4", "6", "--format", "f32", "-i", str(src)],
                           capture_output=True, timeout=300)
    assert first.returncode == 0, first.stderr
    second = subprocess.run(cli + ["flip", "--axis", "y"], input=first.stdout, capture_output=True, timeout=300)
    assert second.returncode == 0, second.stderr
    v = vk.read_volume(src)
    expected = vk.resample(v, (8, 4, 6), vk.DataFormat.FLOAT32)
    vk.flip(expected, "y")
    assert second.stdout == vk.volume_to_bytes(expected)
