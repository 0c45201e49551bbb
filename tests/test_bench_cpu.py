"""CPU: bench.py's reference arm (the unmodified reference's apply_filter on
the host cores) prints the contract's JSON line with the same config as our
arm."""

import json
import subprocess
import sys
from pathlib import Path

import pytest

ROOT = Path(__file__).resolve().parent.parent


@pytest.mark.parametrize("cfg", ["cfg3", "cfg4"])
def test_reference_arm_line(cfg):
    r = subprocess.run([sys.executable, str(ROOT / "bench.py"), "--impl", "reference", "--steps", "1",
                        "--warmup", "0", "--cpu-budget", "0.3", "--config", cfg],
                       capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stderr
    line = json.loads([l for l in r.stdout.splitlines() if l.startswith("{")][-1])
    assert line["impl"] == "reference" and line["value"] > 0
    assert line["higher_is_better"] is True and line["unit"] == "GVox/s"
    cb = line["cpu_baseline"]
    assert cb["value"] == line["value"] and cb["cores"] >= 1
    assert cb["kind"] in ("reference", "port")
    assert line["e2e"]["h2d_bytes_per_step"] == 0
    sys.path.insert(0, str(ROOT))
    import bench

    assert line["config"] == bench.config_dict(cfg, 1)


def test_path_aware_roofline():
    """The roofline's algorithmic work follows the kernel path: kx*ky*kz FMAs
    per voxel dense, kx+ky+kz separable; the bound is the slower of HBM and
    FP32 for that work."""
    sys.path.insert(0, str(ROOT))
    import bench
    import paper_2203_10213_b200 as vk

    k7 = vk.gaussian_kernel(1.5)
    assert bench.algorithmic_fma(k7, "tma") == 343
    assert bench.algorithmic_fma(k7, "separable") == 21
    assert bench.algorithmic_fma(vk.Kernel((9, 1, 3), [1.0] * 27), "separable") == 13
    nvox = 1024 ** 3
    # cfg3 u16 7^3: dense is FP32-bound, separable HBM-bound (4 B per voxel)
    dense = bench.roofline_obj(nvox, 11.05, 2, 343, 6541.5, 1965.0, 148)
    sep = bench.roofline_obj(nvox, 1.65, 2, 21, 6541.5, 1965.0, 148)
    assert dense["bound"] == "fp32" and 0.85 < dense["frac"] < 0.95
    assert sep["bound"] == "hbm" and sep["unit"] == "GB/s"
    assert abs(sep["achieved"] - nvox * 4 / 1.65e-3 / 1e9) < 1.0
    assert abs(sep["frac"] - sep["achieved"] / 6541.5) < 1e-3
    # u8 5^3 separable: 15 FMAs for 2 B per voxel is FP32-bound
    assert bench.roofline_obj(nvox, 1.44, 1, 15, 6541.5, 1965.0, 148)["bound"] == "fp32"
