"""GPU: z-slab sharded ApplyFilter emulated on one GPU.

P "ranks" are P slabs of one volume on cuda:0; the halo exchange uses the
same plan as the NCCL path with in-process copies (no kernel waits on another
kernel).  Each slab runs the real interior / boundary launches with halos, and
the concatenated result must be bit-identical to the unsharded ApplyFilter
(the property the 8-GPU path relies on).  Large-volume tests check
size-independent properties at BASELINE sizes.
"""

import numpy as np
import pytest

import paper_2203_10213_b200 as vk
from paper_2203_10213_b200.shard import ShardedVolume, apply_filter_sharded, plan_halos

pytestmark = pytest.mark.gpu


def _sharded_run(host, fmt, kernel, mode, world, path="auto"):
    import torch

    nz, ny, nx = host.shape
    srcs, dsts = [], []
    for r in range(world):
        s = ShardedVolume((nx, ny, nz), fmt, r, world)
        s.local.upload(np.ascontiguousarray(host[s.z0:s.z1]))
        srcs.append(s)
        dsts.append(ShardedVolume((nx, ny, nz), fmt, r, world))

    def local_exchange(plan, rank, planes, lo, hi):
        # same semantics as exchange_halos, peers' planes read in-process
        halos = {"lo": lo, "hi": hi}
        for t in plan.transfers:
            if t.dst_rank == rank:
                halos[t.side][t.dst_first:t.dst_first + t.count].copy_(
                    srcs[t.src_rank].planes()[t.src_first:t.src_first + t.count])
        for (r, side, slot) in plan.border:
            if r == rank:
                halos[side][slot].zero_()

    vk.set_execution_policy(vk.ExecutionPolicy(filter_path=path))
    try:
        for r in range(world):
            apply_filter_sharded(dsts[r], srcs[r], kernel, mode, exchange=local_exchange)
    finally:
        vk.set_execution_policy(vk.ExecutionPolicy())
    torch.cuda.synchronize()
    return np.concatenate([d.local.to_numpy() for d in dsts])


def _unsharded(host, fmt, kernel, mode, path="auto"):
    src = vk.StructuredVolume.from_numpy(host, fmt)
    dst = vk.StructuredVolume(src.dims, fmt)
    vk.set_execution_policy(vk.ExecutionPolicy(filter_path=path))
    try:
        vk.ApplyFilter(dst, src, kernel, mode)
    finally:
        vk.set_execution_policy(vk.ExecutionPolicy())
    return dst.to_numpy()


@pytest.mark.parametrize("world", [2, 3, 8])
@pytest.mark.parametrize("mode", list(vk.AddressMode))
@pytest.mark.parametrize("fmt,k", [(vk.DataFormat.UINT16, 7), (vk.DataFormat.FLOAT32, 3),
                                   (vk.DataFormat.UINT8, 5), (vk.DataFormat.FLOAT32, 9),
                                   (vk.DataFormat.UINT8, (3, 1, 5)), (vk.DataFormat.FLOAT32, (5, 5, 1)),
                                   (vk.DataFormat.FLOAT32, (3, 1, 3)), (vk.DataFormat.FLOAT32, (1, 5, 5))],
                         ids=lambda v: "x".join(map(str, v)) if isinstance(v, tuple) else str(v))
def test_sharded_bit_identical_to_unsharded(world, mode, fmt, k):
    # K = 9 (rz = 4 > a slab at world 8), and anisotropic kernels: (3,1,5) is
    # cube-padded in the shards too (kz = K); (5,5,1) is padded unsharded only
    # (no halo planes to grow into) and still matches bit for bit
    rng = np.random.default_rng(world * 100 + (k if isinstance(k, int) else sum(k)))
    shape = (40, 24, 64)  # (z, y, x): TMA-eligible rows for every format
    host = (rng.random(shape, dtype=np.float32) if fmt is vk.DataFormat.FLOAT32 else
            rng.integers(0, np.iinfo(fmt.dtype).max + 1, size=shape, dtype=fmt.dtype))
    if isinstance(k, tuple):
        w = rng.random(k[0] * k[1] * k[2])
        kern = vk.Kernel(k, w / w.sum())
    else:
        kern = vk.gaussian_kernel(1.0, k) if k != 5 else vk.box_kernel(5)
    want = _unsharded(host, fmt, kern, mode)
    got = _sharded_run(host, fmt, kern, mode, world)
    assert np.array_equal(got.view(np.uint8), want.view(np.uint8))


@pytest.mark.parametrize("mode", list(vk.AddressMode))
def test_sharded_guarded_f32_sees_nonfinite_halo(mode):
    # (3,1,3) f32 is cube-padded behind an Inf/NaN scan; an Inf / NaN sitting
    # in the planes next to a slab boundary reaches the neighbour only through
    # its halo buffer, whose scan must send that rank to the direct kernel
    rng = np.random.default_rng(17)
    host = rng.random((40, 24, 64), dtype=np.float32)
    host[19, 7, 9] = np.inf   # world 2: rank 0's last plane, rank 1's halo_lo
    host[20, 3, 30] = np.nan  # rank 1's first plane, rank 0's halo_hi
    host[0, 5, 5] = -np.inf   # rank 0's first plane; Wrap: rank 1's halo_hi
    w = rng.random(9)
    kern = vk.Kernel((3, 1, 3), w / w.sum())
    want = _unsharded(host, vk.DataFormat.FLOAT32, kern, mode, "direct")
    got = _sharded_run(host, vk.DataFormat.FLOAT32, kern, mode, 2)
    assert np.array_equal(got.view(np.uint32), want.view(np.uint32))
    fin = host.copy()
    fin[~np.isfinite(fin)] = 0.5
    assert np.array_equal(_sharded_run(fin, vk.DataFormat.FLOAT32, kern, mode, 2),
                          _unsharded(fin, vk.DataFormat.FLOAT32, kern, mode, "direct"))


@pytest.mark.parametrize("world", [2, 3])
@pytest.mark.parametrize("mode", list(vk.AddressMode))
@pytest.mark.parametrize("fmt", [vk.DataFormat.UINT16, vk.DataFormat.FLOAT32])
def test_sharded_separable_large_extent(world, mode, fmt):
    # gaussian_kernel(3.0) is 13^3: rz = 6 halo planes per side, separable
    rng = np.random.default_rng(31 + world)
    host = (rng.random((40, 24, 64), dtype=np.float32) if fmt is vk.DataFormat.FLOAT32 else
            rng.integers(0, 65536, size=(40, 24, 64), dtype=np.uint16))
    kern = vk.gaussian_kernel(3.0)
    want = _unsharded(host, fmt, kern, mode)
    got = _sharded_run(host, fmt, kern, mode, world)
    assert np.array_equal(got.view(np.uint8), want.view(np.uint8))


@pytest.mark.parametrize("world", [2, 3])
@pytest.mark.parametrize("mode", list(vk.AddressMode))
def test_sharded_separable_f32_nonfinite(world, mode):
    # the separable f32 kernel recomputes exactly its Inf / NaN outputs with
    # the dense arithmetic, per launch: an Inf / NaN next to a slab boundary
    # (reached by the neighbour through its halo) still gives bitwise the
    # unsharded result
    rng = np.random.default_rng(23 + world)
    host = rng.random((40, 24, 64), dtype=np.float32)
    host[19, 7, 9] = np.inf
    host[20, 3, 30] = np.nan
    host[0, 5, 5] = -np.inf
    kern = vk.gaussian_kernel(1.0, 5)
    want = _unsharded(host, vk.DataFormat.FLOAT32, kern, mode)
    got = _sharded_run(host, vk.DataFormat.FLOAT32, kern, mode, world)
    assert np.array_equal(got.view(np.uint32), want.view(np.uint32))


@pytest.mark.parametrize("path", ["direct", "exact"])
def test_sharded_other_paths(path):
    rng = np.random.default_rng(4)
    host = rng.integers(0, 65536, size=(11, 9, 13), dtype=np.uint16)
    kern = vk.gaussian_kernel(1.5)  # rz=3 > slab thickness at world 4
    for mode in vk.AddressMode:
        want = _unsharded(host, vk.DataFormat.UINT16, kern, mode, path)
        got = _sharded_run(host, vk.DataFormat.UINT16, kern, mode, 4, path)
        assert np.array_equal(got, want), mode


def test_plan_matches_bench_layout():
    plan = plan_halos(1024, 8, 3, "clamp")
    assert sum(t.count for t in plan.transfers) == 8 * 2 * 3


# ---- full-size, size-independent properties (BASELINE configs) ----

def test_cfg3_1024_u16_delta_is_identity_and_constant_is_fixed():
    import torch

    dims = (1024, 1024, 1024)
    src = vk.synthetic_device(dims, vk.DataFormat.UINT16, seed=3)
    dst = vk.StructuredVolume(src.dims, src.format, data=vk.DeviceBuffer(src.nbytes, zero=False))
    w = np.zeros((7, 7, 7))
    w[3, 3, 3] = 1.0
    vk.ApplyFilter(dst, src, vk.Kernel((7, 7, 7), w))
    assert torch.equal(dst.data.array, src.data.array)
    vk.fill(src, 0.5)
    vk.ApplyFilter(dst, src, vk.gaussian_kernel(1.5))
    # torch has no uint16 reductions: compare the raw 16-bit pattern (32768 = 0x8000)
    assert bool((dst.array().view(torch.int16) == -32768).all())
    del src, dst
    torch.cuda.empty_cache()


def test_cfg4_wrap_laplacian_sums_to_zero_f32():
    """Wrap mode is periodic: sum(out) = sum(w) * sum(in) = 0 for the Laplacian."""
    import torch

    dims = (512, 512, 512)
    src = vk.synthetic_device(dims, vk.DataFormat.FLOAT32, seed=9)
    dst = vk.StructuredVolume(src.dims, src.format)
    vk.ApplyFilter(dst, src, vk.laplacian_kernel(), vk.AddressMode.WRAP)
    total = dst.array().double().sum().item()
    scale = src.array().double().abs().sum().item()
    assert abs(total) <= 1e-6 * scale
    # and box5 in Wrap mode preserves the total
    vk.ApplyFilter(dst, src, vk.box_kernel(5), vk.AddressMode.WRAP)
    s_in = src.array().double().sum().item()
    s_out = dst.array().double().sum().item()
    assert abs(s_out - s_in) <= 1e-5 * abs(s_in)
    del src, dst
    torch.cuda.empty_cache()


def test_cfg2_512_f32_box5_mirror_chunk_vs_oracle():
    """Full 512^3 on the GPU; a z-chunk of it against the oracle (chunked runner)."""
    import torch
    from oracle import vkt_oracle as O

    dims = (512, 512, 512)
    src = vk.synthetic_device(dims, vk.DataFormat.FLOAT32, seed=21)
    dst = vk.StructuredVolume(src.dims, src.format)
    vk.ApplyFilter(dst, src, vk.box_kernel(5), vk.AddressMode.MIRROR)
    host = src.to_numpy()
    for z0, z1 in ((0, 3), (254, 258), (509, 512)):
        want = O.apply_filter(host, 3, O.box_weights(5), "mirror", z_range=(z0, z1))
        got = dst.array()[z0:z1].cpu().numpy()
        d = np.abs(got.astype(np.float64) - want)
        assert np.all(d <= 1e-5 * np.abs(want) + 1e-5)
    del src, dst
    torch.cuda.empty_cache()


# ---- host-buffer entry point (vkt_apply_filter_host): chunked, overlapped ----

@pytest.mark.parametrize("mode", list(vk.AddressMode))
@pytest.mark.parametrize("fmt,k,chunk", [(vk.DataFormat.UINT16, 7, 5), (vk.DataFormat.FLOAT32, 3, 1),
                                         (vk.DataFormat.UINT8, 5, 0), (vk.DataFormat.FLOAT32, 7, 2)])
def test_host_api_bit_identical_to_device(mode, fmt, k, chunk):
    rng = np.random.default_rng(k * 10 + chunk)
    shape = (23, 20, 64)
    host = (rng.random(shape, dtype=np.float32) if fmt is vk.DataFormat.FLOAT32 else
            rng.integers(0, np.iinfo(fmt.dtype).max + 1, size=shape, dtype=fmt.dtype))
    kern = vk.gaussian_kernel(1.0, k) if k != 5 else vk.box_kernel(5)
    want = _unsharded(host, fmt, kern, mode)
    got = vk.apply_filter_host(host, kern, mode, chunk_planes=chunk)
    assert np.array_equal(got.view(np.uint8), want.view(np.uint8))
    got = vk.apply_filter_host(host, kern, mode, chunk_planes=chunk, bounded_memory=True)
    assert np.array_equal(got.view(np.uint8), want.view(np.uint8))
    # a z sub-range writes only those planes
    out = np.zeros_like(host)
    vk.apply_filter_host(host, kern, mode, out=out, z_range=(4, 17), chunk_planes=chunk)
    assert np.array_equal(out[4:17].view(np.uint8), want[4:17].view(np.uint8))
    assert not out[:4].any() and not out[17:].any()


def test_host_api_pinned_large_and_direct_path():
    import torch

    dims = (512, 512, 512)
    src = vk.synthetic_device(dims, vk.DataFormat.UINT16, seed=5)
    dst = vk.StructuredVolume(src.dims, src.format)
    kern = vk.gaussian_kernel(1.5)
    vk.ApplyFilter(dst, src, kern)
    pin_in = torch.empty(src.nbytes, dtype=torch.uint8, pin_memory=True)
    pin_in.copy_(src.data.array)
    pin_out = torch.empty(src.nbytes, dtype=torch.uint8, pin_memory=True)
    host_in = pin_in.numpy().view(np.uint16).reshape(512, 512, 512)
    host_out = pin_out.numpy().view(np.uint16).reshape(512, 512, 512)
    vk.apply_filter_host(host_in, kern, out=host_out)
    assert torch.equal(pin_out, dst.data.array.cpu())
    # generic (non-TMA) kernel through the host path: odd row length
    h = np.random.default_rng(1).integers(0, 65536, size=(9, 7, 13), dtype=np.uint16)
    assert np.array_equal(vk.apply_filter_host(h, kern, "wrap", chunk_planes=2),
                          _unsharded(h, vk.DataFormat.UINT16, kern, vk.AddressMode.WRAP))


def test_host_api_slab_buffers_match_whole_volume():
    """Each 'rank' passes only its halo-extended slab (what range I/O would read)."""
    rng = np.random.default_rng(8)
    host = rng.integers(0, 65536, size=(40, 24, 64), dtype=np.uint16)
    kern = vk.gaussian_kernel(1.5)
    for mode in (vk.AddressMode.CLAMP, vk.AddressMode.MIRROR, vk.AddressMode.BORDER):
        want = _unsharded(host, vk.DataFormat.UINT16, kern, mode)
        got = np.zeros_like(host)
        for z0, z1 in ((0, 13), (13, 27), (27, 40)):
            lo, hi = max(0, z0 - 3), min(40, z1 + 3)
            ext = np.ascontiguousarray(host[lo:hi])
            o = vk.apply_filter_host(ext, kern, mode, z_offset=lo, global_nz=40,
                                     z_range=(z0 - lo, z1 - lo), chunk_planes=4)
            got[z0:z1] = o[z0 - lo:z1 - lo]
        assert np.array_equal(got, want), mode
    # Wrap needs the far planes: a slab without them is rejected, not silently wrong
    with pytest.raises(vk.InvalidArgument):
        vk.apply_filter_host(np.ascontiguousarray(host[0:16]), kern, "wrap", z_offset=0, global_nz=40,
                             z_range=(0, 13))


@pytest.mark.parametrize("bounded", [False, True])
@pytest.mark.parametrize("mode", list(vk.AddressMode))
@pytest.mark.parametrize("kd,chunk", [((7, 7, 7), 16), ((9, 9, 9), 16), ((3, 3, 3), 40), ((5, 5, 5), 0)])
def test_host_api_ramped_chunks_and_halo_reuse(mode, kd, chunk, bounded):
    """Ramped chunk schedule (C/4, C/2, C.., C/2, C/4) with the low halo of each
    chunk copied device-to-device from the previous chunk's input: chunks
    smaller than the 2*rz halo included (9^3 kernel, 4-plane ramp chunks)."""
    rng = np.random.default_rng(sum(kd) + chunk)
    host = rng.integers(0, 65536, size=(70, 18, 64), dtype=np.uint16)
    w = rng.random(kd[0] * kd[1] * kd[2])
    kern = vk.Kernel(kd, w / w.sum())
    want = _unsharded(host, vk.DataFormat.UINT16, kern, mode)
    got = vk.apply_filter_host(host, kern, mode, chunk_planes=chunk, bounded_memory=bounded)
    assert np.array_equal(got, want)
    out = np.zeros_like(host)
    vk.apply_filter_host(host, kern, mode, out=out, z_range=(9, 61), chunk_planes=chunk,
                         bounded_memory=bounded)
    assert np.array_equal(out[9:61], want[9:61])
