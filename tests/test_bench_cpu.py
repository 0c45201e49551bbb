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
