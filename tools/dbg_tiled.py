import sys; sys.path.insert(0, '.'); sys.path.insert(0, 'tests')
import numpy as np
import paper_2203_10213_b200 as vk
from oracle import vkt_oracle as O
from test_gpu_parity import run_filter
for fmt, k, mode in [(1,3,'clamp'), (1,3,'border'), (2,7,'clamp'), (3,7,'clamp'), (3,3,'wrap')]:
    rng = np.random.default_rng(1000 * fmt + k)
    dims = (80, 37, 23)
    stored = (rng.random((dims[2], dims[1], dims[0]), dtype=np.float32) if fmt == 3 else
              rng.integers(0, np.iinfo(O.DTYPE[fmt]).max + 1, size=dims[::-1], dtype=O.DTYPE[fmt]))
    w = O.gaussian_weights(1.0, k) if k != 5 else O.box_weights(5)
    want = O.apply_filter(stored, fmt, w, mode).astype(np.float64)
    got = run_filter(stored, fmt, w, mode).astype(np.float64)
    bad = np.abs(got - want) > (1 if fmt != 3 else 1e-4)
    zz, yy, xx = np.nonzero(bad)
    print(fmt, k, mode, "bad", bad.sum(), "x", np.unique(xx)[:40], "y", np.unique(yy)[:40], "z", np.unique(zz)[:30])
