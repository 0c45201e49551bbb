"""CPU, multi-process: z-slab halo plan + exchange over torch.distributed (gloo).

The same ``exchange_halos`` that runs over NCCL on the GPUs runs here over
gloo with CPU tensors at world sizes 2 and 3.  Each rank checks that its
halos hold exactly the address-mapped global planes, and that filtering its
halo-extended slab (oracle as the checker) reproduces the unsharded result
bit-for-bit — the property the device path relies on.
"""

import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2203_10213_b200.filters import AddressMode
from paper_2203_10213_b200.shard import exchange_halos, map_plane, plan_halos, slab_bounds


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _global_volume(nx, ny, nz):
    rng = np.random.default_rng(nx * 1000 + ny * 10 + nz)
    return rng.integers(0, 65536, size=(nz, ny, nx), dtype=np.uint16)


def _worker(rank, world, port, configs, errq):
    try:
        os.environ["MASTER_ADDR"] = "127.0.0.1"
        os.environ["MASTER_PORT"] = str(port)
        dist.init_process_group("gloo", rank=rank, world_size=world)
        from oracle import vkt_oracle as O

        for (nx, ny, nz), kz, mode in configs:
            vol = _global_volume(nx, ny, nz)
            rz = kz // 2
            z0, z1 = slab_bounds(nz, world, rank)
            plane_bytes = nx * ny * 2
            local = torch.from_numpy(np.ascontiguousarray(vol[z0:z1]).view(np.uint8).reshape(z1 - z0, plane_bytes))
            lo = torch.full((rz, plane_bytes), 0xAB, dtype=torch.uint8)
            hi = torch.full((rz, plane_bytes), 0xAB, dtype=torch.uint8)
            plan = plan_halos(nz, world, rz, mode)
            exchange_halos(plan, rank, local, lo, hi)
            # 1) halo content == address-mapped global planes (zeros for Border)
            for side, buf, first in (("lo", lo, z0 - rz), ("hi", hi, z1)):
                got = buf.numpy().view(np.uint16).reshape(rz, ny, nx)
                for s in range(rz):
                    m = map_plane(first + s, nz, AddressMode.coerce(mode))
                    want = np.zeros((ny, nx), np.uint16) if m is None else vol[m]
                    assert np.array_equal(got[s], want), (rank, side, s, mode)
            # 2) filtering the extended slab == the unsharded result
            ext = np.concatenate([lo.numpy().view(np.uint16).reshape(rz, ny, nx), vol[z0:z1],
                                  hi.numpy().view(np.uint16).reshape(rz, ny, nx)])
            w = O.gaussian_weights(1.0, kz) if kz > 1 else np.ones((1, 1, 1))
            part = O.apply_filter(ext, 2, w, mode, z_range=(rz, rz + z1 - z0), workers=1)
            full = O.apply_filter(vol, 2, w, mode, z_range=(z0, z1), workers=1)
            assert np.array_equal(part, full), (rank, mode, kz)
        dist.barrier()
        dist.destroy_process_group()
    except BaseException as e:  # surface the failure to the parent
        errq.put(f"rank {rank}: {type(e).__name__}: {e}")
        raise


def _run(world, configs):
    ctx = mp.get_context("spawn")
    errq = ctx.SimpleQueue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, configs, errq)) for r in range(world)]
    for p in procs:
        p.start()
    for p in procs:
        p.join(timeout=240)
    errors = []
    while not errq.empty():
        errors.append(errq.get())
    for p in procs:
        if p.is_alive():
            p.kill()
            errors.append("timeout")
    assert not errors and all(p.exitcode == 0 for p in procs), errors


MODES = ["clamp", "wrap", "mirror", "border"]


def test_exchange_world2():
    _run(2, [((9, 7, 12), k, m) for k in (3, 7) for m in MODES])


def test_exchange_world3_thin_slabs():
    # nz=5 over 3 ranks with rz=3: halos thicker than a slab, served by several ranks
    _run(3, [((6, 5, 5), 7, m) for m in MODES] + [((6, 5, 13), 5, m) for m in MODES])


def test_plan_is_minimal_for_interior_ranks():
    plan = plan_halos(1024, 8, 3, "clamp")
    sends, recvs, local, zeros = plan.for_rank(3)
    assert len(recvs) == 2 and all(t.count == 3 for t in recvs)
    assert not local and not zeros
    # ring for wrap
    plan = plan_halos(1024, 8, 1, "wrap")
    _, recvs0, _, _ = plan.for_rank(0)
    assert {t.src_rank for t in recvs0} == {7, 1}
    # border: edge ranks get zero planes, no traffic
    plan = plan_halos(64, 4, 2, "border")
    _, recvs0, local0, zeros0 = plan.for_rank(0)
    assert len(zeros0) == 2 and {t.src_rank for t in recvs0} == {1} and not local0


def test_plan_rejects_empty_slabs():
    from paper_2203_10213_b200.errors import InvalidArgument

    with pytest.raises(InvalidArgument):
        plan_halos(3, 4, 1, "clamp")
