"""GPU: ApplyFilter / FillRange captured into a CUDA graph and replayed.

Small volumes are launch-bound (cfg1, 256^3 u8: ~15 us of host time per call
against ~40 us of kernel), so the C ABI must stay capture-safe: no device
queries or allocations that invalidate a capture (the scratch pool allocates
stream-ordered).  The replayed results must equal the eager ones.
"""

import numpy as np
import pytest

import paper_2203_10213_b200 as vk

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("fmt,k,mode", [(vk.DataFormat.UINT8, 3, "clamp"), (vk.DataFormat.UINT16, 5, "wrap"),
                                        (vk.DataFormat.FLOAT32, 3, "mirror"), (vk.DataFormat.FLOAT32, 7, "border")])
def test_graph_replay_equals_eager(fmt, k, mode):
    import torch

    src = vk.synthetic_device((256, 64, 40), fmt, seed=5)
    eager = vk.StructuredVolume(src.dims, fmt)
    kern = vk.gaussian_kernel(1.0, k)
    vk.ApplyFilter(eager, src, kern, mode)  # warm-up outside the capture
    out = vk.StructuredVolume(src.dims, fmt)
    side = torch.cuda.Stream()
    side.wait_stream(torch.cuda.current_stream())
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g, stream=side):
        vk.FillRange(out, ((0, 0, 0), (256, 64, 40)), 0.25)
        vk.ApplyFilter(out, src, kern, mode)
    torch.cuda.current_stream().wait_stream(side)
    out.data.raw.zero_()
    g.replay()
    torch.cuda.synchronize()
    assert np.array_equal(out.to_numpy().view(np.uint8), eager.to_numpy().view(np.uint8))
