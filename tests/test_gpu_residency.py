"""GPU: residency of the reference-compatible volumes (ManagedBuffer,
Device.CPU / EMULATED_DEVICE) and device selection.

Host-resident volumes keep the reference's numpy ``array()`` semantics while
every algorithm computes on the B200; results must be byte-identical to the
same calls on HBM-resident volumes.
"""

import numpy as np
import pytest

import paper_2203_10213_b200 as vk
import paper_2203_10213_b200.vkt as vkt
from oracle import vkt_oracle as O

pytestmark = pytest.mark.gpu


@pytest.fixture(autouse=True)
def _reset():
    vkt.set_execution_policy(vkt.ExecutionPolicy())
    yield
    vkt.set_execution_policy(vkt.ExecutionPolicy())
    vkt.emulated_device.set_capacity(None)


def _random(rng, dims, fmt):
    v = vkt.StructuredVolume(dims, fmt)
    a = v.array()
    assert isinstance(a, np.ndarray)  # host residency: a numpy view
    a[...] = (rng.random(a.shape, dtype=np.float32) if fmt is vkt.DataFormat.FLOAT32
              else rng.integers(0, np.iinfo(a.dtype).max + 1, size=a.shape, dtype=a.dtype))
    return v


@pytest.mark.parametrize("fmt", list(vk.DataFormat))
@pytest.mark.parametrize("mode", ["clamp", "wrap"])
def test_host_resident_filter_equals_device_filter(fmt, mode):
    rng = np.random.default_rng(3)
    v = _random(rng, (45, 17, 13), fmt)
    stored = v.array().copy()
    k = vk.gaussian_kernel(1.0, 5)
    dev_src = vk.StructuredVolume.from_numpy(stored, fmt)
    dev_dst = vk.StructuredVolume(dev_src.dims, fmt)
    vk.ApplyFilter(dev_dst, dev_src, k, mode)
    vkt.apply_filter(v, k) if mode == "clamp" else vk.apply_filter(v, k, mode)
    assert v.on_host and v.data.migration_count == 0
    assert np.array_equal(v.array().view(np.uint8), dev_dst.to_numpy().view(np.uint8))
    ok = np.abs(v.array().astype(np.float64) - O.apply_filter(stored, fmt.value, k.weights, mode)).max()
    assert ok <= (1 if fmt is not vk.DataFormat.FLOAT32 else 1e-5)


def test_host_resident_fill_writes_through_pinned_memory():
    v = vkt.StructuredVolume((64, 64, 64), vkt.DataFormat.UINT8)
    vkt.fill_range(v, vkt.box3i((1, 1, 1), (63, 63, 63)), 1.0)
    arr = v.array()
    assert int((arr == 255).sum()) == 62**3 and int((arr == 0).sum()) == 64**3 - 62**3
    vkt.fill(v, 0.5)
    assert np.all(v.array() == 128)
    assert v.get_value((3, 4, 5)) == 128 / 255


def test_migration_follows_policy_and_counts():
    v = vkt.StructuredVolume((8, 8, 8), vkt.DataFormat.UINT8)
    vkt.fill(v, 0.5)
    assert v.data.migration_count == 0 and v.on_host
    vkt.set_execution_policy(vkt.ExecutionPolicy(device=vkt.Device.EMULATED_DEVICE))
    vkt.fill(v, 0.25)
    assert v.data.migration_count == 1 and not v.on_host
    assert vkt.emulated_device.used_bytes >= 512
    a = v.array()
    assert a.is_cuda and int(a[0, 0, 0]) == 64
    vkt.apply_filter(v, vkt.gaussian_kernel(1.0, 3))  # in place on the device: no migration
    assert v.data.migration_count == 1
    vkt.set_execution_policy(vkt.ExecutionPolicy())
    assert np.all(v.array() == 64) and v.data.migration_count == 2 and v.on_host


def test_emulated_capacity_raises_allocation_failure():
    vkt.set_execution_policy(vkt.ExecutionPolicy(device=vkt.Device.EMULATED_DEVICE))
    vkt.emulated_device.set_capacity(vkt.emulated_device.used_bytes + 1000)
    with pytest.raises(vkt.errors.AllocationFailure):
        vkt.StructuredVolume((16, 16, 16), vkt.DataFormat.UINT8)
    vkt.StructuredVolume((8, 8, 8), vkt.DataFormat.UINT8)


def test_host_resident_transforms_and_mapped_arrays():
    rng = np.random.default_rng(8)
    v = _random(rng, (20, 9, 6), vkt.DataFormat.UINT16)
    v.mapping = vk.VoxelMapping(-1.0, 3.0)
    stored = v.array().copy()
    vkt.flip(v, "x")
    assert np.array_equal(v.array(), stored[:, :, ::-1])
    vkt.flip(v, "x")
    out = vkt.resample(v, (10, 9, 6))
    assert out.on_host and out.array().shape == (6, 9, 10)
    m = v.mapped_array()
    assert m.dtype == np.float64 and np.array_equal(m, -1.0 + (stored / 65535.0) * 4.0)
    n = v.normalized_array()
    assert n.min() >= 0.0 and n.max() <= 1.0
    vkt.clahe_equalize(v, vkt.ClaheParams((2, 1, 1), 64, 4.0))
    assert v.on_host and v.array().dtype == np.uint16


def test_device_index_policy_uses_that_device():
    """a volume on a non-current device must filter correctly (the
    C ABI makes the stream's device current for the call)."""
    import torch

    n = torch.cuda.device_count()
    idx = n - 1
    vk.set_execution_policy(vk.ExecutionPolicy(device_index=idx))
    try:
        rng = np.random.default_rng(1)
        stored = rng.integers(0, 256, size=(9, 8, 64), dtype=np.uint8)
        src = vk.StructuredVolume.from_numpy(stored)
        dst = vk.StructuredVolume(src.dims, src.format)
        assert src.data.device.index == idx
        with torch.cuda.device(0):
            vk.ApplyFilter(dst, src, vk.gaussian_kernel(1.0, 3))
            vk.fill_range(src, ((0, 0, 0), (4, 4, 4)), 0.5)
        got = dst.to_numpy().astype(int)
        want = O.apply_filter(stored, 1, vk.gaussian_kernel(1.0, 3).weights, "clamp").astype(int)
        assert np.abs(got - want).max() <= 1
        assert np.all(src.to_numpy()[:4, :4, :4] == 128)
    finally:
        vk.set_execution_policy(vk.ExecutionPolicy())
