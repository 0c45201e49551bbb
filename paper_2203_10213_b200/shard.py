"""z-slab sharding of ApplyFilter across the GPUs of one box.

The reference parallelises one process's ``apply_filter`` over ≤64 z-slabs on
a thread pool (pkg/src/vkt/execution.py:162-170, ops/filters.py:82-95); the
fixed (dz, dy, dx) tap order makes the result independent of the split
(filters.py:87-88).  Here each rank (one process per GPU) owns the planes
``[floor(p*nz/P), floor((p+1)*nz/P))`` of the volume and needs, per side,
``rz = kz//2`` halo planes: the global planes just outside its slab after the
address mode has been applied.  Those planes are fetched with NCCL send/recv
(through ``torch.distributed``) on a high-priority comm stream while the
interior kernel (output planes ``[rz, n-rz)``, which need no halo) runs on
the compute stream; two thin boundary launches follow the halos on the comm
stream, beside the interior.
Every output voxel sees the same taps in the same order as on one GPU, so
sharded results are bit-identical to unsharded ones.

The halo plan is pure host logic and works for any P, any rz (including halos
thicker than a slab, served by several ranks) and every address mode:
  Wrap   - the halo of rank 0 comes from rank P-1 and vice versa (a ring)
  Mirror - reflected planes, served by whichever rank owns them
  Clamp  - edge planes (a local copy at ranks 0 and P-1)
  Border - zero planes (stored 0), no communication
"""

from __future__ import annotations

from dataclasses import dataclass
from typing import Optional

from .errors import InvalidArgument
from .filters import AddressMode, Kernel, _flags, launch, make_args
from .execution import get_execution_policy, timed
from .volume import DataFormat, DeviceBuffer, StructuredVolume


def slab_bounds(nz: int, world: int, rank: int) -> tuple[int, int]:
    """Planes [z0, z1) owned by ``rank`` of ``world`` (balanced, contiguous)."""
    return (rank * nz) // world, ((rank + 1) * nz) // world


def map_plane(g: int, n: int, mode: AddressMode) -> Optional[int]:
    """Global plane index after the address mode (None = Border zero plane).

    Same closed forms as the device ``map_index`` (csrc/common.cuh) and as
    np.pad's edge / wrap / symmetric / constant modes for any overhang.
    """
    if 0 <= g < n:
        return g
    if mode is AddressMode.CLAMP:
        return 0 if g < 0 else n - 1
    if mode is AddressMode.WRAP:
        return g % n
    if mode is AddressMode.MIRROR:
        m = g % (2 * n)
        return m if m < n else 2 * n - 1 - m
    return None


@dataclass(frozen=True)
class Transfer:
    """Planes ``src_rank[src_first : src_first+count]`` -> ``dst_rank``'s halo."""

    src_rank: int
    src_first: int
    dst_rank: int
    side: str          # "lo" | "hi"
    dst_first: int
    count: int


@dataclass(frozen=True)
class HaloPlan:
    nz: int
    world: int
    rz: int
    mode: AddressMode
    transfers: tuple[Transfer, ...]
    border: tuple[tuple[int, str, int], ...]  # (rank, side, halo slot) zero planes

    def for_rank(self, rank: int):
        sends = [t for t in self.transfers if t.src_rank == rank and t.dst_rank != rank]
        recvs = [t for t in self.transfers if t.dst_rank == rank and t.src_rank != rank]
        local = [t for t in self.transfers if t.src_rank == rank and t.dst_rank == rank]
        zeros = [(side, slot) for (r, side, slot) in self.border if r == rank]
        return sends, recvs, local, zeros


def plan_halos(nz: int, world: int, rz: int, mode) -> HaloPlan:
    """Deterministic global exchange plan; every rank computes the same one."""
    mode = AddressMode.coerce(mode)
    if world < 1 or nz < world:
        raise InvalidArgument(f"cannot split {nz} planes over {world} ranks")
    bounds = [slab_bounds(nz, world, p) for p in range(world)]

    def owner(m: int) -> tuple[int, int]:
        for q, (a, b) in enumerate(bounds):
            if a <= m < b:
                return q, m - a
        raise AssertionError(m)

    transfers: list[Transfer] = []
    border: list[tuple[int, str, int]] = []
    for p, (z0, z1) in enumerate(bounds):
        for side, first in (("lo", z0 - rz), ("hi", z1)):
            run: Optional[list[int]] = None  # [src_rank, src_first, dst_first, count]
            for slot in range(rz):
                m = map_plane(first + slot, nz, mode)
                if m is None:
                    border.append((p, side, slot))
                    if run:
                        transfers.append(Transfer(run[0], run[1], p, side, run[2], run[3]))
                        run = None
                    continue
                q, j = owner(m)
                if run and run[0] == q and run[1] + run[3] == j:
                    run[3] += 1
                    continue
                if run:
                    transfers.append(Transfer(run[0], run[1], p, side, run[2], run[3]))
                run = [q, j, slot, 1]
            if run:
                transfers.append(Transfer(run[0], run[1], p, side, run[2], run[3]))
    return HaloPlan(nz, world, rz, mode, tuple(transfers), tuple(border))


def exchange_halos(plan: HaloPlan, rank: int, local_planes, halo_lo, halo_hi, group=None) -> None:
    """Fill this rank's halo buffers according to ``plan``.

    ``local_planes``/``halo_lo``/``halo_hi`` are 2-D byte tensors
    (planes, plane_bytes) on this rank's device (CUDA + NCCL) or on the CPU
    (gloo, for the multi-process CPU tests).  Runs on the current stream.
    """
    import torch.distributed as dist

    sends, recvs, local, zeros = plan.for_rank(rank)
    halos = {"lo": halo_lo, "hi": halo_hi}
    for side, slot in zeros:
        halos[side][slot].zero_()
    for t in local:
        halos[t.side][t.dst_first:t.dst_first + t.count].copy_(
            local_planes[t.src_first:t.src_first + t.count])
    if not sends and not recvs:
        return
    # Every rank walks the global transfer list in the same order, so the
    # k-th message between a (src, dst) pair is posted as the k-th on both
    # sides; the index doubles as the tag for backends that match on tags.
    ops = []
    for tag, t in enumerate(plan.transfers):
        if t.src_rank == t.dst_rank:
            continue
        if t.src_rank == rank:
            ops.append(dist.P2POp(dist.isend, local_planes[t.src_first:t.src_first + t.count],
                                  t.dst_rank, group, tag))
        if t.dst_rank == rank:
            ops.append(dist.P2POp(dist.irecv, halos[t.side][t.dst_first:t.dst_first + t.count],
                                  t.src_rank, group, tag))
    for w in dist.batch_isend_irecv(ops):
        w.wait()


def exchange_halos_host_staged(plan: HaloPlan, rank: int, local_planes, halo_lo, halo_hi,
                               group=None) -> None:
    """``exchange_halos`` for backends without device P2P (gloo): the planes
    this rank sends are staged to host memory, exchanged, and the received
    halos copied back.  Used by the multi-process tests that run several ranks
    on one GPU, where NCCL's spinning P2P kernels must not share a device."""
    sends, recvs, _local, _zeros = plan.for_rank(rank)
    need = sorted({(t.src_first, t.count) for t in sends})
    host_planes = local_planes.cpu() if need else local_planes[:0].cpu()
    h_lo, h_hi = halo_lo.cpu(), halo_hi.cpu()
    exchange_halos(plan, rank, host_planes, h_lo, h_hi, group)
    halo_lo.copy_(h_lo)
    halo_hi.copy_(h_hi)


class ShardedVolume:
    """This rank's z-slab of a global volume, plus its halo buffers."""

    def __init__(self, global_dims, fmt: DataFormat, rank: int, world: int, *,
                 mapping=(0.0, 1.0), cell_size=(1.0, 1.0, 1.0), local: StructuredVolume = None,
                 device=None):
        self.global_dims = tuple(int(d) for d in global_dims)
        nx, ny, nz = self.global_dims
        self.rank, self.world = rank, world
        self.z0, self.z1 = slab_bounds(nz, world, rank)
        if self.z1 <= self.z0:
            raise InvalidArgument(f"rank {rank} of {world} owns no planes of nz={nz}")
        self.format = fmt
        if local is None:
            local = StructuredVolume((nx, ny, self.z1 - self.z0), fmt, cell_size, mapping,
                                     data=DeviceBuffer(nx * ny * (self.z1 - self.z0) * fmt.bytes_per_cell,
                                                       device=device, zero=False))
        elif tuple(local.dims) != (nx, ny, self.z1 - self.z0):
            raise InvalidArgument("local slab has the wrong extents")
        self.local = local
        self._halo: dict[int, tuple] = {}

    @property
    def plane_bytes(self) -> int:
        nx, ny, _ = self.global_dims
        return nx * ny * self.format.bytes_per_cell

    def planes(self):
        return self.local.data.array.view(self.local.dims.z, self.plane_bytes)

    def halo_buffers(self, rz: int):
        if rz not in self._halo:
            lo = DeviceBuffer(rz * self.plane_bytes, device=self.local.data.device, zero=True)
            hi = DeviceBuffer(rz * self.plane_bytes, device=self.local.data.device, zero=True)
            self._halo[rz] = (lo, hi)
        return self._halo[rz]


_comm_streams: dict = {}


def _comm_stream(device):
    import torch

    s = _comm_streams.get(device)
    if s is None:
        s = torch.cuda.Stream(device=device, priority=-1)
        _comm_streams[device] = s
    return s


@timed("ApplyFilterSharded")
def apply_filter_sharded(dst: ShardedVolume, src: ShardedVolume, kernel: Kernel,
                         address_mode=AddressMode.CLAMP, group=None, exchange=None,
                         kernel_events: Optional[list] = None,
                         phase_events: Optional[dict] = None) -> None:
    """Sharded ApplyFilter: halo exchange overlapped with the interior kernel.

    ``exchange(plan, rank, planes, halo_lo, halo_hi)`` defaults to the NCCL /
    torch.distributed ``exchange_halos``; tests substitute an in-process
    copy.  ``kernel_events``, if given, receives one (start, end) CUDA event
    pair around the main (interior) launch, for the bench's roofline;
    ``phase_events`` (a dict) receives (start, end) pairs on the comm stream
    under "exchange" (the halo exchange) and "boundary" (the boundary
    launches), for the bench's per-rank breakdown.
    """
    import torch

    exchange = exchange or (lambda *a: exchange_halos(*a, group=group))

    def timed_launch(a):
        if kernel_events is None:
            launch(a, int(compute.cuda_stream))
            return
        e0 = torch.cuda.Event(enable_timing=True)
        e1 = torch.cuda.Event(enable_timing=True)
        e0.record(compute)
        launch(a, int(compute.cuda_stream))
        e1.record(compute)
        kernel_events.append((e0, e1))

    mode = AddressMode.coerce(address_mode)
    if dst.global_dims != src.global_dims or dst.rank != src.rank or dst.format is not src.format:
        raise InvalidArgument("dst and src shards differ in layout")
    nx, ny, nz = src.global_dims
    n = src.local.dims.z
    rz = kernel.radius.z
    flags = _flags(get_execution_policy())
    dev = src.local.data.device
    compute = torch.cuda.current_stream(dev)
    common = dict(dims=(nx, ny, n), fmt=src.format, mapping=src.local.mapping, kernel=kernel,
                  mode=mode, z_offset=src.z0, global_nz=nz, flags=flags)

    if src.world == 1 or rz == 0:
        a, _k = make_args(dst.local.data_ptr(), src.local.data_ptr(), **common)
        timed_launch(a)
        return

    plan = plan_halos(nz, src.world, rz, mode)
    lo, hi = src.halo_buffers(rz)
    comm = _comm_stream(dev)
    comm.wait_stream(compute)  # src planes are final

    def mark(key):
        if phase_events is None:
            return None
        ev = torch.cuda.Event(enable_timing=True)
        ev.record(comm)
        return (key, ev)

    def close(opened):
        if opened is not None:
            ev = torch.cuda.Event(enable_timing=True)
            ev.record(comm)
            phase_events.setdefault(opened[0], []).append((opened[1], ev))

    opened = mark("exchange")
    with torch.cuda.stream(comm), torch.cuda.nvtx.range("vkt halo exchange"):
        exchange(plan, src.rank, src.planes(), lo.array.view(rz, src.plane_bytes),
                 hi.array.view(rz, src.plane_bytes))
    close(opened)
    halo_ptrs = dict(halo_lo=lo.data_ptr(), halo_hi=hi.data_ptr())
    if n > 2 * rz:
        a, _k = make_args(dst.local.data_ptr(), src.local.data_ptr(), **common, **halo_ptrs,
                          out_z_begin=rz, out_z_end=n - rz)
        timed_launch(a)
        ranges = ((0, rz), (n - rz, n))
    else:
        ranges = ((0, n),)
    # The boundary planes run on the comm stream right behind the exchange,
    # beside the interior launch: their CTAs fill the SMs the interior's tail
    # leaves idle (measured on one GPU, cfg3 slab at P = 8: +1.2% over a
    # single launch, against +4.5% when they ran after the interior;
    # tools/shard_overhead.py).  Disjoint output planes; the compute stream
    # joins the comm stream before anything else touches dst.
    opened = mark("boundary")
    for b, e in ranges:  # NVTX: vkt_apply_filter ranges from the library
        a, _k = make_args(dst.local.data_ptr(), src.local.data_ptr(), **common, **halo_ptrs,
                          out_z_begin=b, out_z_end=e)
        launch(a, int(comm.cuda_stream))
    close(opened)
    compute.wait_stream(comm)
    lo.tensor.record_stream(comm)
    hi.tensor.record_stream(comm)
