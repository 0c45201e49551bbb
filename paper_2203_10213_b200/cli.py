"""Command line tool for the B200 ApplyFilter path.

Mirrors the reference CLI's subcommands on this path (pkg/src/vkt/cli.py):

    python -m paper_2203_10213_b200 filter --gaussian 1.0 --ksize 3 -i in.vkt -o out.vkt
    python -m paper_2203_10213_b200 filter --kernel-file k.txt [--mode wrap] < in.vkt > out.vkt
    python -m paper_2203_10213_b200 fill --value 0.5 [--roi X0 Y0 Z0 X1 Y1 Z1] -i in.vkt
    python -m paper_2203_10213_b200 clahe --bricks 2 2 2 [--bins 256] [--clip 4] -i in.vkt
    python -m paper_2203_10213_b200 resample --dims X Y Z [--format f32] [--range LO HI] -i in.vkt
    python -m paper_2203_10213_b200 flip --axis y -i in.vkt
    python -m paper_2203_10213_b200 info -i in.vkt
    python -m paper_2203_10213_b200 raw-import --dims X Y Z --format u8 -i raw.bin
    python -m paper_2203_10213_b200 bench [--size 128] [--repeat 3]

Volumes travel as VKTVOL01 bytes over files or standard streams.  Exit codes
are the reference's: 0 success, 1 usage error, 2 data error with the line
``error: <ErrorName>: <message>`` on stderr (cli.py:547-564), which the TS
bindings parse (cli.ts:38).  A failing invocation never leaves a partial
output file (cli.py:209-225).  ``filter`` with both ``-i`` and ``-o`` files
streams the volume through the GPU out of core (``io.filter_file``), so
volumes larger than host RAM and HBM work.  New: ``--mode`` selects the
address mode (the reference always clamps).
"""

from __future__ import annotations

import argparse
import math
import os
import sys
import tempfile
import time
from pathlib import Path

from . import io as vio
from .errors import InvalidArgument, IoFailure, VktError
from .execution import ExecutionPolicy, set_execution_policy


class _Parser(argparse.ArgumentParser):
    """Usage errors exit 1, not argparse's 2 (cli.py:35-42)."""

    def error(self, message):
        self.print_usage(sys.stderr)
        print(f"{self.prog}: error: {message}", file=sys.stderr)
        raise SystemExit(1)


def _io_args(p, output=True):
    p.add_argument("-i", "--input", help="input volume path (default: standard input)")
    if output:
        p.add_argument("-o", "--output", help="output path (default: standard output)")


def _build_parser() -> _Parser:
    parser = _Parser(prog="vkt-b200", description="B200-native ApplyFilter / Fill for volkit volumes")
    parser.add_argument("--device", choices=["cuda"], default="cuda",
                        help="device space (the B200; there is no CPU path)")
    parser.add_argument("--workers", type=int, default=0,
                        help="accepted for compatibility; the GPU grid decides")
    parser.add_argument("--timings", action="store_true",
                        help="print per-algorithm wall times to standard error")
    sub = parser.add_subparsers(dest="command", parser_class=_Parser, required=True)

    p = sub.add_parser("info", help="describe a volume")
    _io_args(p)

    p = sub.add_parser("fill", help="fill cells with a value")
    _io_args(p)
    p.add_argument("--value", type=float, required=True)
    p.add_argument("--roi", type=int, nargs=6, metavar=("X0", "Y0", "Z0", "X1", "Y1", "Z1"))

    p = sub.add_parser("filter", help="correlate with a kernel (ApplyFilter)")
    _io_args(p)
    p.add_argument("--gaussian", type=float, metavar="SIGMA")
    p.add_argument("--ksize", type=int, help="kernel extent for --gaussian (odd)")
    p.add_argument("--kernel-file", help="text file: first line 'X Y Z', then weights")
    p.add_argument("--mode", choices=["clamp", "wrap", "mirror", "border"], default="clamp",
                   help="address mode (the reference always clamps)")
    p.add_argument("--chunk-planes", type=int, default=0, help="z-planes per streamed chunk")

    p = sub.add_parser("clahe", help="contrast limited adaptive histogram equalization")
    _io_args(p)
    p.add_argument("--bricks", type=int, nargs=3, required=True, metavar=("X", "Y", "Z"))
    p.add_argument("--bins", type=int, default=256)
    p.add_argument("--clip", type=float, default=math.inf,
                   help="clip limit as a multiple of the uniform bin height (inf = off)")

    p = sub.add_parser("resample", help="resample onto a new structured grid")
    _io_args(p)
    p.add_argument("--dims", type=int, nargs=3, required=True, metavar=("X", "Y", "Z"))
    p.add_argument("--format", choices=["u8", "u16", "f32"])
    p.add_argument("--range", type=float, nargs=2, metavar=("LO", "HI"))

    p = sub.add_parser("flip", help="mirror along an axis")
    _io_args(p)
    p.add_argument("--axis", choices=["x", "y", "z"], required=True)

    p = sub.add_parser("raw-import", help="wrap a headerless raw payload")
    _io_args(p)
    p.add_argument("--dims", type=int, nargs=3, required=True, metavar=("X", "Y", "Z"))
    p.add_argument("--format", choices=["u8", "u16", "f32"], required=True)
    p.add_argument("--range", type=float, nargs=2, default=[0.0, 1.0], metavar=("LO", "HI"))
    p.add_argument("--cell-size", type=float, nargs=3, default=[1.0, 1.0, 1.0],
                   metavar=("X", "Y", "Z"))

    p = sub.add_parser("bench", help="time the ApplyFilter cases of the reference bench")
    p.add_argument("-o", "--output", help="report path (default: standard output)")
    p.add_argument("--size", type=int, default=128)
    p.add_argument("--subgrids", type=int, default=64, help="accepted for compatibility")
    p.add_argument("--bench-workers", type=int, default=8)
    p.add_argument("--repeat", type=int, default=3)
    return parser


# -- stream helpers (cli.py:191-233) -----------------------------------------

def _read_volume_arg(args):
    if getattr(args, "input", None):
        return vio.read_volume(args.input)
    payload = sys.stdin.buffer.read()
    if not payload:
        raise IoFailure("no input volume: pass -i PATH or pipe volume bytes")
    return vio.volume_from_bytes(payload)


def _write_bytes_out(path, payload: bytes) -> None:
    if not path:
        sys.stdout.buffer.write(payload)
        sys.stdout.buffer.flush()
        return
    target = Path(path)
    fd, tmp = tempfile.mkstemp(dir=str(target.parent) or ".", prefix=target.name + ".")
    try:
        with os.fdopen(fd, "wb") as fh:
            fh.write(payload)
        os.replace(tmp, target)
    except BaseException:
        try:
            os.unlink(tmp)
        except OSError:
            pass
        raise


def _write_volume_out(args, volume) -> None:
    _write_bytes_out(getattr(args, "output", None), vio.volume_to_bytes(volume))


def _kernel(args):
    from .filters import Kernel, gaussian_kernel

    if (args.gaussian is None) == (args.kernel_file is None):
        raise InvalidArgument("pass exactly one of --gaussian or --kernel-file")
    if args.gaussian is not None:
        return gaussian_kernel(args.gaussian, args.ksize)
    try:
        text = Path(args.kernel_file).read_text().split()
    except OSError as e:
        raise IoFailure(str(e)) from e
    dims = [int(v) for v in text[:3]]
    weights = [float(v) for v in text[3:]]
    return Kernel(dims, weights)


# -- commands ----------------------------------------------------------------

def _cmd_info(args) -> int:
    if getattr(args, "input", None):
        dims, fmt, cell_size, mapping = vio.read_header(args.input)
    else:
        dims, fmt, cell_size, mapping = vio.parse_header(sys.stdin.buffer.read(vio.HEADER_SIZE))
    lines = [
        "type: structured",
        f"dims: {dims.x}x{dims.y}x{dims.z}",
        f"format: {fmt.short_name}",
        f"cell size: {cell_size[0]:g} {cell_size[1]:g} {cell_size[2]:g}",
        f"range: {mapping.lo:g} {mapping.hi:g}",
        f"cells: {dims.x * dims.y * dims.z}",
    ]
    _write_bytes_out(getattr(args, "output", None), ("\n".join(lines) + "\n").encode())
    return 0


def _cmd_fill(args) -> int:
    from .fill import fill, fill_range
    from .geom import box3i

    volume = _read_volume_arg(args)
    if args.roi:
        fill_range(volume, box3i(args.roi[:3], args.roi[3:]), args.value)
    else:
        fill(volume, args.value)
    _write_volume_out(args, volume)
    return 0


def _cmd_filter(args) -> int:
    from .filters import apply_filter

    kernel = _kernel(args)
    if args.input and args.output:
        vio.filter_file(args.input, args.output, kernel, args.mode, chunk_planes=args.chunk_planes)
        return 0
    volume = _read_volume_arg(args)
    apply_filter(volume, kernel, args.mode)
    _write_volume_out(args, volume)
    return 0


def _cmd_clahe(args) -> int:
    from .clahe import ClaheParams, clahe_equalize

    volume = _read_volume_arg(args)
    clahe_equalize(volume, ClaheParams(tuple(args.bricks), args.bins, args.clip))
    _write_volume_out(args, volume)
    return 0


def _cmd_resample(args) -> int:
    from .transforms import resample
    from .volume import DataFormat, VoxelMapping

    volume = _read_volume_arg(args)
    fmt = DataFormat.parse(args.format) if args.format else None
    mapping = VoxelMapping(*args.range) if args.range else None
    _write_volume_out(args, resample(volume, args.dims, fmt, mapping))
    return 0


def _cmd_flip(args) -> int:
    from .transforms import flip

    volume = _read_volume_arg(args)
    flip(volume, args.axis)
    _write_volume_out(args, volume)
    return 0


def _cmd_raw_import(args) -> int:
    if getattr(args, "input", None):
        try:
            payload = Path(args.input).read_bytes()
        except OSError as e:
            raise IoFailure(str(e)) from e
    else:
        payload = sys.stdin.buffer.read()
    volume = vio.load_raw(payload, args.dims, args.format, args.cell_size, tuple(args.range))
    _write_volume_out(args, volume)
    return 0


def _cmd_bench(args) -> int:
    """The ApplyFilter-path cases of the reference bench (bench.py:88-146):
    gaussian_filter (gaussian_kernel(1.0, 3) on synthetic_structured(size),
    setup copy outside the timer) and fillrange, best of `repeat`, device
    time.  One device executes both the "serial" and the "parallel" plan,
    so both columns report the same measurement."""
    import torch

    from .fill import fill_range
    from .filters import apply_filter, gaussian_kernel
    from .synthetic import synthetic_structured

    volume = synthetic_structured(args.size)
    kernel = gaussian_kernel(1.0, 3)

    def best(fn, setup):
        b = math.inf
        for _ in range(max(1, args.repeat)):
            ctx = setup() if setup else None
            torch.cuda.synchronize()
            t0 = time.perf_counter()
            fn(ctx)
            torch.cuda.synchronize()
            b = min(b, time.perf_counter() - t0)
        return b

    cases = [
        ("fillrange", lambda _: fill_range(volume, volume.bounds, 0.5), None),
        ("gaussian_filter", lambda v: apply_filter(v, kernel), volume.copy),
    ]
    lines = []
    for name, fn, setup in cases:
        best(fn, setup)  # warm-up
        t = best(fn, setup)
        lines.append(f"bench: case={name} serial_s={t:.6f} parallel_s={t:.6f} "
                     f"workers={args.bench_workers} effective_workers=1")
    _write_bytes_out(getattr(args, "output", None), ("\n".join(lines) + "\n").encode())
    return 0


_COMMANDS = {
    "info": _cmd_info,
    "fill": _cmd_fill,
    "filter": _cmd_filter,
    "clahe": _cmd_clahe,
    "resample": _cmd_resample,
    "flip": _cmd_flip,
    "raw-import": _cmd_raw_import,
    "bench": _cmd_bench,
}


def main(argv=None) -> int:
    parser = _build_parser()
    try:
        args = parser.parse_args(argv)
    except SystemExit as e:
        return int(e.code or 0)
    set_execution_policy(ExecutionPolicy(worker_count=args.workers, print_timings=args.timings))
    try:
        return _COMMANDS[args.command](args)
    except VktError as e:
        print(f"error: {e.name}: {e}", file=sys.stderr)
        return 2
    except OSError as e:
        print(f"error: IoFailure: {e}", file=sys.stderr)
        return 2


if __name__ == "__main__":
    sys.exit(main())
