"""VKTVOL01 volume files feeding the B200.

Same on-disk format as the reference (pkg/src/vkt/io.py:3-26): the 8-byte
magic ``VKTVOL01``, a volume-type byte (0 = structured), dims 3 x u32, the
format code u8, cell size 3 x f32, mapping lo/hi 2 x f32 — 42 bytes — then
the raw cells x-fastest.  Only structured volumes are on the ApplyFilter path.

What changes is where the bytes go: payloads stream through page-locked
staging buffers straight into / out of HBM in large chunks (file reads
overlap the host-to-device copies), and ``filter_file`` filters a volume file
of ANY size out of core: z-chunks plus their halo planes are read,
filtered by ``vkt_apply_filter_host`` and written, with reading, GPU work and
writing of consecutive chunks overlapped.  The header is 42 bytes and planes
are contiguous, so a z-slab is one seek + one read.
"""

from __future__ import annotations

import io as _io
import os
import struct
import tempfile
from contextlib import contextmanager
from concurrent.futures import ThreadPoolExecutor
from pathlib import Path
from typing import BinaryIO, Union

import numpy as np

from .errors import (
    BadMagic,
    EmptyRange,
    InvalidArgument,
    IoFailure,
    NotSeekable,
    RangeOutOfBounds,
    SizeMismatch,
    TruncatedPayload,
    UnknownFormatCode,
)
from .execution import timed
from .geom import Box3i, Vec3i, coerce_box, full_box, ivec3
from .volume import DataFormat, DeviceBuffer, StructuredVolume, VoxelMapping

MAGIC = b"VKTVOL01"
_STRUCTURED = 0
_HIERARCHICAL = 1
_HEADER = struct.Struct("<3IB3f2f")                  # after magic + type byte (io.py:59)
HEADER_SIZE = len(MAGIC) + 1 + _HEADER.size          # 42 bytes (io.py:65)
_STAGE = 64 << 20                                     # staging chunk (bytes)

Source = Union[str, os.PathLike, bytes, bytearray, BinaryIO]


# -- header ------------------------------------------------------------------

def _new_file_mode(target: Path) -> int:
    """Mode a plain open() would give ``target``: the existing file's, else
    0o666 minus the umask (mkstemp's 0o600 would make outputs owner-only)."""
    try:
        return target.stat().st_mode & 0o7777
    except OSError:
        mask = os.umask(0)
        os.umask(mask)
        return 0o666 & ~mask


@contextmanager
def atomic_output(path):
    """Binary file that replaces ``path`` only once the block completes: the
    bytes go to a sibling temporary file that is renamed into place, so a
    failed command never leaves a partial output (the reference CLI's
    contract, cli.py:209-225)."""
    target = Path(path)
    mode = _new_file_mode(target)
    handle = tempfile.NamedTemporaryFile(mode="w+b", dir=str(target.parent) or ".",
                                         prefix=f".{target.name}.", delete=False)
    done = False
    try:
        with handle:
            yield handle
            handle.flush()
        os.chmod(handle.name, mode)
        os.replace(handle.name, target)
        done = True
    finally:
        if not done:
            try:
                os.unlink(handle.name)
            except OSError:
                pass


def pack_header(dims, fmt: DataFormat, cell_size, mapping) -> bytes:
    d = ivec3(dims)
    m = VoxelMapping.coerce(mapping)
    return MAGIC + bytes([_STRUCTURED]) + _HEADER.pack(d.x, d.y, d.z, fmt.value, *map(float, cell_size),
                                                       m.lo, m.hi)


def parse_header(raw: bytes):
    """(dims, fmt, cell_size, mapping) of a structured-volume header."""
    if len(raw) < len(MAGIC):
        raise TruncatedPayload(f"expected {len(MAGIC)} bytes of magic, got {len(raw)}")
    if raw[:len(MAGIC)] != MAGIC:
        raise BadMagic(f"expected {MAGIC!r}, got {raw[:len(MAGIC)]!r}")
    if len(raw) < len(MAGIC) + 1:
        raise TruncatedPayload("missing volume type")
    vtype = raw[len(MAGIC)]
    if vtype == _HIERARCHICAL:
        raise InvalidArgument("hierarchical volumes are not on the ApplyFilter path (structured only)")
    if vtype != _STRUCTURED:
        raise UnknownFormatCode(f"unknown volume type {vtype}")
    if len(raw) < HEADER_SIZE:
        raise TruncatedPayload(f"expected {HEADER_SIZE} header bytes, got {len(raw)}")
    f = _HEADER.unpack(raw[len(MAGIC) + 1:HEADER_SIZE])
    if f[3] not in (1, 2, 3):
        raise UnknownFormatCode(f"unknown data format code {f[3]}")
    return Vec3i(f[0], f[1], f[2]), DataFormat(f[3]), tuple(f[4:7]), VoxelMapping(f[7], f[8])


class _Stream:
    """Binary stream over a path, bytes or a file object (DataSource, io.py:68-145)."""

    def __init__(self, src: Source, mode: str = "rb"):
        self.owned = False
        if isinstance(src, (str, os.PathLike)):
            try:
                self.f = open(src, mode)
            except OSError as e:
                raise IoFailure(str(e)) from e
            self.owned = True
        elif isinstance(src, (bytes, bytearray)):
            self.f = _io.BytesIO(bytes(src))
        else:
            self.f = src
        self.seekable = getattr(self.f, "seekable", lambda: False)()

    def read_exact(self, n: int, what: str) -> bytes:
        data = self.f.read(n)
        if len(data) != n:
            raise TruncatedPayload(f"expected {n} bytes of {what}, got {len(data)}")
        return data

    def readinto_exact(self, view: memoryview, what: str) -> None:
        got = 0
        while got < len(view):
            n = self.f.readinto(view[got:])
            if not n:
                raise TruncatedPayload(f"expected {len(view)} bytes of {what}, got {got}")
            got += n

    def close(self):
        if self.owned:
            self.f.close()

    def __enter__(self):
        return self

    def __exit__(self, *exc):
        self.close()


def read_header(src: Source):
    with _Stream(src) as s:
        return parse_header(s.read_exact(HEADER_SIZE, "structured header"))


# -- pinned staging ----------------------------------------------------------

def _pinned(nbytes: int):
    import torch

    return torch.empty(max(nbytes, 1), dtype=torch.uint8, pin_memory=torch.cuda.is_available())


def _upload_stream(stream: _Stream, dst_u8, nbytes: int, what: str) -> None:
    """File bytes -> device bytes through two alternating pinned chunks."""
    import torch

    bufs = [_pinned(min(_STAGE, nbytes)) for _ in range(2)]
    done = [None, None]
    cs = torch.cuda.current_stream(dst_u8.device)
    off = 0
    i = 0
    while off < nbytes:
        n = min(_STAGE, nbytes - off)
        b = bufs[i % 2]
        if done[i % 2] is not None:
            done[i % 2].synchronize()       # the copy out of this buffer finished
        stream.readinto_exact(memoryview(b.numpy())[:n], what)
        dst_u8[off:off + n].copy_(b[:n], non_blocking=True)
        ev = torch.cuda.Event()
        ev.record(cs)
        done[i % 2] = ev
        off += n
        i += 1
    cs.synchronize()


def _download_stream(src_u8, f, nbytes: int) -> None:
    """Device bytes -> file through two alternating pinned chunks."""
    import torch

    bufs = [_pinned(min(_STAGE, nbytes)) for _ in range(2)]
    cs = torch.cuda.current_stream(src_u8.device)
    events = []
    offs = list(range(0, nbytes, _STAGE))
    # enqueue the first copy, then overlap writing chunk i with copying i+1
    for i, off in enumerate(offs):
        n = min(_STAGE, nbytes - off)
        b = bufs[i % 2]  # its previous chunk (i-2) was written out at iteration i-1
        b[:n].copy_(src_u8[off:off + n], non_blocking=True)
        ev = torch.cuda.Event()
        ev.record(cs)
        events.append(ev)
        if i >= 1:
            prev = offs[i - 1]
            pn = min(_STAGE, nbytes - prev)
            events[i - 1].synchronize()
            f.write(memoryview(bufs[(i - 1) % 2].numpy())[:pn])
    if offs:
        events[-1].synchronize()
        last = offs[-1]
        f.write(memoryview(bufs[(len(offs) - 1) % 2].numpy())[:nbytes - last])


# -- whole-volume serialization ----------------------------------------------

@timed("ReadVolume")
def read_volume(src: Source) -> StructuredVolume:
    """VKTVOL01 structured volume -> device volume (io.py:203-236)."""
    with _Stream(src) as s:
        dims, fmt, cell_size, mapping = parse_header(s.read_exact(HEADER_SIZE, "structured header"))
        nbytes = dims.x * dims.y * dims.z * fmt.bytes_per_cell
        vol = StructuredVolume(dims, fmt, cell_size, mapping, data=DeviceBuffer(nbytes, zero=False))
        _upload_stream(s, vol.data.array, nbytes, "cell payload")
        return vol


@timed("WriteVolume")
def write_volume(dst: Union[str, os.PathLike, BinaryIO], volume: StructuredVolume) -> None:
    """Device volume -> VKTVOL01 (io.py:164-194)."""
    if not isinstance(volume, StructuredVolume):
        raise InvalidArgument(f"cannot serialize {type(volume).__name__}")
    owned = isinstance(dst, (str, os.PathLike))
    try:
        f = open(dst, "wb") if owned else dst
    except OSError as e:
        raise IoFailure(str(e)) from e
    try:
        f.write(pack_header(volume.dims, volume.format, volume.cell_size, volume.mapping))
        _download_stream(volume.data.array, f, volume.nbytes)
        f.flush()
    finally:
        if owned:
            f.close()


def volume_to_bytes(volume: StructuredVolume) -> bytes:
    sink = _io.BytesIO()
    write_volume(sink, volume)
    return sink.getvalue()


def volume_from_bytes(payload: bytes) -> StructuredVolume:
    return read_volume(payload)


def load_raw(src: Source, dims, fmt, cell_size=(1.0, 1.0, 1.0), mapping=(0.0, 1.0)) -> StructuredVolume:
    """Headerless payload whose length must match exactly (io.py:257-276)."""
    dims = ivec3(dims, "dims")
    fmt = fmt if isinstance(fmt, DataFormat) else DataFormat.parse(fmt)
    expected = dims.x * dims.y * dims.z * fmt.bytes_per_cell
    with _Stream(src) as s:
        payload = s.f.read()
    if len(payload) != expected:
        raise SizeMismatch(f"raw payload holds {len(payload)} bytes, "
                           f"{dims.x}x{dims.y}x{dims.z} {fmt.short_name} needs {expected}")
    vol = StructuredVolume(dims, fmt, cell_size, mapping, data=DeviceBuffer(expected, zero=False))
    vol.fill_bytes(payload)
    return vol


# -- range-partial I/O -------------------------------------------------------

def _read_box_host(s: _Stream, dims, fmt, roi: Box3i) -> np.ndarray:
    """Cells of `roi` as a host (z, y, x) array; whole rows / planes are
    coalesced into single reads (the reference reads row by row, io.py:298-328)."""
    bpc = fmt.bytes_per_cell
    d = roi.dims
    out = np.empty((d.z, d.y, d.x), dtype=fmt.dtype)
    x0, y0, z0 = roi.lower
    row_b = dims.x * bpc
    plane_b = row_b * dims.y
    if d.x == dims.x and d.y == dims.y:                    # z-slab: one read
        s.f.seek(HEADER_SIZE + z0 * plane_b)
        s.readinto_exact(memoryview(out.reshape(-1).view(np.uint8)), "z-slab")
    elif d.x == dims.x:                                     # whole rows: one read per plane
        for k in range(d.z):
            s.f.seek(HEADER_SIZE + (z0 + k) * plane_b + y0 * row_b)
            s.readinto_exact(memoryview(out[k].reshape(-1).view(np.uint8)), "rows")
    else:
        for k in range(d.z):
            for j in range(d.y):
                s.f.seek(HEADER_SIZE + ((z0 + k) * dims.y + y0 + j) * row_b + x0 * bpc)
                s.readinto_exact(memoryview(out[k, j].view(np.uint8)), "row")
    return out


def read_range(src: Source, roi) -> StructuredVolume:
    """Exactly the cells of `roi` as a device volume (io.py:298-328)."""
    with _Stream(src) as s:
        if not s.seekable:
            raise NotSeekable("range reads need a seekable source")
        dims, fmt, cell_size, mapping = parse_header(s.read_exact(HEADER_SIZE, "structured header"))
        roi = coerce_box(roi)
        if roi.is_empty:
            raise EmptyRange(f"roi {tuple(roi.lower)}..{tuple(roi.upper)} selects no cells")
        b = full_box(dims)
        if not all(b.lower[a] <= roi.lower[a] and roi.upper[a] <= b.upper[a] for a in range(3)):
            raise RangeOutOfBounds(f"roi exceeds volume dims {tuple(dims)}")
        host = _read_box_host(s, dims, fmt, roi)
        return StructuredVolume.from_numpy(host, fmt, cell_size, mapping)


def write_range(dst: Union[str, os.PathLike, BinaryIO], volume: StructuredVolume, first_cell) -> None:
    """Overwrite the sub-box at `first_cell` of an existing file (io.py:331-357)."""
    owned = isinstance(dst, (str, os.PathLike))
    try:
        f = open(dst, "r+b") if owned else dst
    except OSError as e:
        raise IoFailure(str(e)) from e
    try:
        if not f.seekable():
            raise NotSeekable("range writes need a seekable destination")
        f.seek(0)
        dims, fmt, _, _ = parse_header(f.read(HEADER_SIZE))
        first = ivec3(first_cell, "first cell")
        if volume.format is not fmt:
            raise InvalidArgument(f"volume format {volume.format.short_name} differs from file "
                                  f"format {fmt.short_name}")
        end = [first[a] + volume.dims[a] for a in range(3)]
        if min(first) < 0 or any(end[a] > dims[a] for a in range(3)):
            raise RangeOutOfBounds(f"sub-box at {tuple(first)} with dims {tuple(volume.dims)} "
                                   f"exceeds file dims {tuple(dims)}")
        host = volume.to_numpy()
        bpc = fmt.bytes_per_cell
        row_b = dims.x * bpc
        for k in range(volume.dims.z):
            if volume.dims.x == dims.x:
                f.seek(HEADER_SIZE + ((first.z + k) * dims.y + first.y) * row_b)
                f.write(host[k].tobytes())
                continue
            for j in range(volume.dims.y):
                f.seek(HEADER_SIZE + ((first.z + k) * dims.y + first.y + j) * row_b + first.x * bpc)
                f.write(host[k, j].tobytes())
        f.flush()
    finally:
        if owned:
            f.close()


# -- out-of-core filtering ---------------------------------------------------

@timed("FilterFile")
def filter_file(src, dst, kernel, address_mode=None, *, chunk_planes: int = 0) -> None:
    """ApplyFilter a VKTVOL01 file into another, any size, never holding it all.

    The reference loads the volume, filters in place and writes it back
    (cli.py:359-375).  Here z-chunks of the input (plus their address-mapped
    halo planes, read directly from the file) are filtered by the B200
    host-buffer pipeline and written at their offset in the output; reading
    chunk c+1 and writing chunk c-1 overlap the GPU work on chunk c.  The
    output is written to a temporary file and renamed into place, so a
    failure never leaves a partial output (cli.py:209-225).
    """
    from .filters import AddressMode, apply_filter_host
    from .shard import map_plane

    mode = AddressMode.CLAMP if address_mode is None else AddressMode.coerce(address_mode)
    src = Path(src)
    dst = Path(dst)
    with _Stream(src) as s:
        header = s.read_exact(HEADER_SIZE, "structured header")
    dims, fmt, _cell, mapping = parse_header(header)
    nx, ny, nz = dims
    bpc = fmt.bytes_per_cell
    plane_b = nx * ny * bpc
    if src.stat().st_size < HEADER_SIZE + plane_b * nz:
        raise TruncatedPayload(f"{src} holds fewer than {plane_b * nz} payload bytes")
    rz = kernel.radius.z
    C = chunk_planes if chunk_planes > 0 else max(8, (256 << 20) // plane_b)
    C = min(C, nz)
    chunks = [(z0, min(z0 + C, nz)) for z0 in range(0, nz, C)]

    with atomic_output(dst) as out_f, open(src, "rb") as in_f:
        out_f.write(header)
        out_f.truncate(HEADER_SIZE + plane_b * nz)

        # two pinned slab and output buffers in rotation: chunk c reads into
        # slab[c % 2] (chunk c-2 was filtered before c-1 started) and
        # filters into out[c % 2] (chunk c-2's write finished before
        # chunk c-1's write was queued)
        slab_bufs = [_pinned(C * plane_b) for _ in range(min(2, len(chunks)))]
        out_bufs = [_pinned(C * plane_b) for _ in range(min(2, len(chunks)))]

        def view(buf, n):
            return buf.numpy()[:n * plane_b].view(fmt.dtype).reshape(n, ny, nx)

        def read_chunk(c, z0, z1):
            slab = view(slab_bufs[c % 2], z1 - z0)
            in_f.seek(HEADER_SIZE + z0 * plane_b)
            _Stream(in_f).readinto_exact(memoryview(slab.reshape(-1).view(np.uint8)), "z-slab")
            halos = []
            for first in (z0 - rz, z1):
                if rz == 0:
                    halos.append(None)
                    continue
                h = np.zeros((rz, ny, nx), dtype=fmt.dtype)
                for t in range(rz):
                    m = map_plane(first + t, nz, mode)
                    if m is None:
                        continue  # Border: stored 0
                    in_f.seek(HEADER_SIZE + m * plane_b)
                    _Stream(in_f).readinto_exact(memoryview(h[t].reshape(-1).view(np.uint8)), "halo")
                halos.append(h)
            return slab, halos

        def write_chunk(z0, out):
            out_f.seek(HEADER_SIZE + z0 * plane_b)
            out_f.write(memoryview(out.reshape(-1).view(np.uint8)))

        with ThreadPoolExecutor(max_workers=1) as reader, ThreadPoolExecutor(max_workers=1) as writer:
            pending_read = reader.submit(read_chunk, 0, *chunks[0])
            pending_write = None
            for c, (z0, z1) in enumerate(chunks):
                slab, halos = pending_read.result()
                if c + 1 < len(chunks):
                    pending_read = reader.submit(read_chunk, c + 1, *chunks[c + 1])
                out = view(out_bufs[c % 2], z1 - z0)
                apply_filter_host(slab, kernel, mode, fmt=fmt, mapping=tuple(mapping), out=out,
                                  z_offset=z0, global_nz=nz, halo_lo=halos[0], halo_hi=halos[1])
                if pending_write is not None:
                    pending_write.result()
                pending_write = writer.submit(write_chunk, z0, out)
            if pending_write is not None:
                pending_write.result()

