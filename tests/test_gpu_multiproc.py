"""GPU, multi-process: the sharded device path in real separate processes.

Two ranks share cuda:0 (only one GPU is available); each runs the real
interior / boundary kernel launches of ``apply_filter_sharded`` on its own
slab.  The halo transport is ``exchange_halos_host_staged`` over gloo,
because NCCL's P2P kernels spin on their peer and must not share one GPU.
Every rank's slab must be bit-identical to the unsharded result.
"""

import os
import socket

import numpy as np
import pytest
import torch.multiprocessing as mp

pytestmark = pytest.mark.gpu


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _worker(rank, world, port, errq):
    try:
        os.environ["MASTER_ADDR"] = "127.0.0.1"
        os.environ["MASTER_PORT"] = str(port)
        import torch
        import torch.distributed as dist

        import paper_2203_10213_b200 as vk
        from paper_2203_10213_b200.shard import (ShardedVolume, apply_filter_sharded,
                                                 exchange_halos_host_staged)

        torch.cuda.set_device(0)
        dist.init_process_group("gloo", rank=rank, world_size=world)
        for fmt, k, mode in ((vk.DataFormat.UINT16, vk.gaussian_kernel(1.5), "clamp"),
                             (vk.DataFormat.FLOAT32, vk.laplacian_kernel(), "wrap"),
                             (vk.DataFormat.UINT8, vk.box_kernel(5), "mirror"),
                             (vk.DataFormat.FLOAT32, vk.gaussian_kernel(1.0, 3), "border")):
            dims = (128, 48, 37)
            whole = vk.synthetic_device(dims, fmt, seed=3)
            want_vol = vk.StructuredVolume(whole.dims, fmt)
            vk.ApplyFilter(want_vol, whole, k, mode)
            src = ShardedVolume(dims, fmt, rank, world)
            dst = ShardedVolume(dims, fmt, rank, world)
            gen = vk.synthetic_device(dims, fmt, seed=3, z_offset=src.z0, local_nz=src.z1 - src.z0)
            src.local.swap_storage(gen)
            apply_filter_sharded(dst, src, k, mode, exchange=lambda *a: exchange_halos_host_staged(*a))
            torch.cuda.synchronize()
            want = want_vol.to_numpy()[src.z0:src.z1]
            got = dst.local.to_numpy()
            assert np.array_equal(got.view(np.uint8), want.view(np.uint8)), (rank, fmt, mode)
        dist.barrier()
        dist.destroy_process_group()
    except BaseException as e:
        errq.put(f"rank {rank}: {type(e).__name__}: {e}")
        raise


@pytest.mark.parametrize("world", [2, 3])
def test_sharded_processes_bit_identical(world):
    ctx = mp.get_context("spawn")
    errq = ctx.SimpleQueue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, errq)) for r in range(world)]
    for p in procs:
        p.start()
    for p in procs:
        p.join(timeout=300)
    errors = []
    while not errq.empty():
        errors.append(errq.get())
    for p in procs:
        if p.is_alive():
            p.kill()
            errors.append("timeout")
    assert not errors and all(p.exitcode == 0 for p in procs), errors
