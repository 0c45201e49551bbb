"""Small ApplyFilter launches of every tiled kernel family for compute-sanitizer
(racecheck / synccheck / memcheck): u8/u16/f32 x K = 3/5/7/9 x the four
address modes, on a volume with interior and edge tiles, plus a sharded
boundary launch (halo buffers) and a pitched (unaligned rows) shape.

  compute-sanitizer --tool racecheck python tools/sanitize_cases.py
"""
import sys
from pathlib import Path

import numpy as np

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import paper_2203_10213_b200 as vk  # noqa: E402
from oracle import vkt_oracle as O  # noqa: E402

only = sys.argv[1:]  # optional subset of formats
rng = np.random.default_rng(0)
n = 0
for fmt in (vk.DataFormat.UINT8, vk.DataFormat.UINT16, vk.DataFormat.FLOAT32):
    if only and fmt.short_name not in only:
        continue
    for dims in ((272, 40, 14), (137, 19, 9)):  # 3 x-tiles x 2-3 y-tiles; unaligned rows
        shape = dims[::-1]
        host = (rng.random(shape, dtype=np.float32) if fmt is vk.DataFormat.FLOAT32 else
                rng.integers(0, np.iinfo(fmt.dtype).max + 1, size=shape, dtype=fmt.dtype))
        src = vk.StructuredVolume.from_numpy(host, fmt)
        dst = vk.StructuredVolume(src.dims, fmt)
        for k in (3, 5, 7, 9):
            kern = vk.gaussian_kernel(1.0, k)
            for mode in vk.AddressMode:
                vk.ApplyFilter(dst, src, kern, mode)
                n += 1
                if k == 3 and dims[0] == 137:  # checked against the oracle too
                    got = dst.to_numpy().astype(np.float64)
                    want = O.apply_filter(host, fmt.value, kern.weights, mode.name.lower()).astype(np.float64)
                    assert np.abs(got - want).max() <= (1 if fmt is not vk.DataFormat.FLOAT32 else 1e-5), (fmt, mode)
print(f"sanitize cases: {n} launches ok")
