import os
import sys
from pathlib import Path

import numpy as np
import pytest

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))
GOLDEN = ROOT / "tests" / "golden"


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200) and the built library")


def cuda_ok() -> bool:
    try:
        import torch

        return torch.cuda.is_available()
    except Exception:
        return False


def pytest_collection_modifyitems(config, items):
    if cuda_ok():
        return
    skip = pytest.mark.skip(reason="no CUDA device visible")
    for item in items:
        if "gpu" in item.keywords:
            item.add_marker(skip)


MODE_NAMES = ("wrap", "mirror", "clamp", "border")


def load_filter_cases():
    """Golden ApplyFilter fixtures generated from the reference (oracle/make_golden.py)."""
    z = np.load(GOLDEN / "filter_cases.npz")
    keys = sorted({k.split("/")[0] for k in z.files})
    out = []
    for k in keys:
        meta = z[f"{k}/meta"]
        out.append(dict(
            key=k,
            name=str(z[f"{k}/name"]),
            input=z[f"{k}/input"],
            output=z[f"{k}/output"],
            weights=z[f"{k}/weights"],
            fmt=int(meta[0]),
            lo=float(meta[1]),
            hi=float(meta[2]),
            mode=MODE_NAMES[int(meta[3])],
        ))
    return out


def load_fill_cases():
    z = np.load(GOLDEN / "fill_cases.npz")
    keys = sorted({k.split("/")[0] for k in z.files})
    out = []
    for k in keys:
        s = z[f"{k}/spec"]
        out.append(dict(
            key=k, input=z[f"{k}/input"], output=z[f"{k}/output"], fmt=int(s[0]),
            lo=float(s[1]), hi=float(s[2]), lower=tuple(int(v) for v in s[3:6]),
            upper=tuple(int(v) for v in s[6:9]), value=float(s[9]),
        ))
    return out


def within_contract(got: np.ndarray, ref: np.ndarray, fmt: int):
    """BASELINE.md §5 parity contract for the fast (f32-accumulate) path.

    ints: |got - ref| <= 1 LSB.  f32: |got - ref| <= 1e-5*|ref| + 1e-5
    (rtol 1e-5 from the north star plus the reference's own 1e-5 absolute
    criterion, pkg/tests/test_acceptance.py:65-70).
    Returns (ok, n_differing, max_abs_diff).
    """
    if fmt == 3:
        g = got.astype(np.float64)
        r = ref.astype(np.float64)
        d = np.abs(g - r)
        ok = bool(np.all(d <= 1e-5 * np.abs(r) + 1e-5))
        return ok, int((d > 0).sum()), float(d.max(initial=0.0))
    d = np.abs(got.astype(np.int64) - ref.astype(np.int64))
    return bool(d.max(initial=0) <= 1), int((d > 0).sum()), float(d.max(initial=0))
