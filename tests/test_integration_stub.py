"""GPU: the reference-side ctypes binding of INTEGRATION.md §2, executed.

The code block of INTEGRATION.md §2 is written, as documented, to
``vkt/ops/_b200.py`` inside a copy of the UNMODIFIED reference package
(baseline/_ref/vkt, installed by build()), with only the library path filled
in.  A subprocess then filters and fills reference volumes through the stub
and compares with the reference's own apply_filter / fill_range.
"""

import os
import re
import shutil
import subprocess
import sys
from pathlib import Path

import pytest

ROOT = Path(__file__).resolve().parent.parent
REF_PKG = ROOT / "baseline" / "_ref" / "vkt"
LIB = ROOT / "paper_2203_10213_b200" / "libvkt_b200.so"

DRIVER = r'''
import numpy as np, vkt
from vkt.ops import _b200
rng = np.random.default_rng(5)
for fmt in (vkt.DataFormat.UINT8, vkt.DataFormat.UINT16, vkt.DataFormat.FLOAT32):
    v = vkt.StructuredVolume((37, 21, 12), fmt, (1, 1, 1), (0.0, 1.0))
    a = v.array()
    a[...] = (rng.random(a.shape, dtype=np.float32) if fmt is vkt.DataFormat.FLOAT32
              else rng.integers(0, np.iinfo(a.dtype).max + 1, size=a.shape, dtype=a.dtype))
    ref = v.copy()
    k = vkt.gaussian_kernel(1.0, 3)
    vkt.apply_filter(ref, k)                 # the reference itself (filters.py:69-95)
    _b200.apply_filter(v, k)                 # the documented stub -> libvkt_b200.so
    g, r = v.array().astype(np.float64), ref.array().astype(np.float64)
    if fmt is vkt.DataFormat.FLOAT32:
        assert np.all(np.abs(g - r) <= 1e-5 * np.abs(r)), float(np.abs(g - r).max())
    else:
        assert np.abs(g - r).max() <= 1, float(np.abs(g - r).max())
    roi = vkt.box3i((3, 2, 1), (30, 19, 11))
    want = v.copy()
    vkt.fill_range(want, roi, 0.25)
    from vkt.volume import quantize
    _b200.fill_range(v, roi, quantize(0.25, v.format, v.mapping))
    assert v.data.to_bytes() == want.data.to_bytes()
try:
    _b200.apply_filter(v, vkt.Kernel((3, 3, 3), np.zeros(27)), mode=9)
    raise SystemExit("bad mode accepted")
except vkt.errors.InvalidArgument:
    pass
print("stub ok")
'''


def _stub_source() -> str:
    text = (ROOT / "INTEGRATION.md").read_text()
    section = text[text.index("## 2."):text.index("## 3.")]
    blocks = re.findall(r"```python\n(.*?)```", section, re.S)
    assert len(blocks) == 1, "INTEGRATION.md §2 must hold exactly one python block"
    return blocks[0].replace('ctypes.CDLL("libvkt_b200.so")', f'ctypes.CDLL("{LIB}")')


def test_stub_block_is_documented():
    src = _stub_source()
    compile(src, "vkt/ops/_b200.py", "exec")
    for name in ("def apply_filter", "def fill_range", "vkt_apply_filter", "vkt_fill_box"):
        assert name in src


@pytest.mark.gpu
def test_stub_runs_inside_the_reference_package(tmp_path):
    if not (REF_PKG / "__init__.py").exists():
        pytest.skip("baseline/_ref not installed (run __graft_entry__.build() where /root/reference exists)")
    shutil.copytree(REF_PKG, tmp_path / "vkt")
    (tmp_path / "vkt" / "ops" / "_b200.py").write_text(_stub_source())
    env = dict(os.environ, PYTHONPATH=str(tmp_path))
    r = subprocess.run([sys.executable, "-c", DRIVER], cwd=tmp_path, env=env, capture_output=True,
                       text=True, timeout=600)
    assert r.returncode == 0 and "stub ok" in r.stdout, r.stdout + r.stderr
