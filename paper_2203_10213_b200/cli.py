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
output file (cli.py:209-225; io.atomic_output).  ``filter`` with both ``-i`` and ``-o`` files
streams the volume through the GPU out of core (``io.filter_file``), so
volumes larger than host RAM and HBM work.  New: ``--mode`` selects the
address mode (the reference always clamps).
"""

from __future__ import annotations

import argparse
import math
import sys
from pathlib import Path

import numpy as np

from . import io as vio
from .errors import InvalidArgument, IoFailure, VktError
from .execution import ExecutionPolicy, set_execution_policy


class _Parser(argparse.ArgumentParser):
    """argparse with the reference's usage-error status: 1 instead of 2
    (cli.py:35-42); the usage line and message still go to stderr."""

    USAGE_ERROR = 1

    def error(self, message):
        self.exit(self.USAGE_ERROR, f"{self.format_usage()}{self.prog}: error: {message}\n")


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


# -- input / output (same streams and messages as cli.py:191-233) -----------

def _input_bytes(args) -> bytes:
    """The raw input payload: the -i file, else standard input."""
    path = getattr(args, "input", None)
    if not path:
        return sys.stdin.buffer.read()
    try:
        return Path(path).read_bytes()
    except OSError as exc:
        raise IoFailure(str(exc)) from exc


def _read_volume_arg(args):
    path = getattr(args, "input", None)
    if path:
        return vio.read_volume(path)
    payload = _input_bytes(args)
    if payload:
        return vio.volume_from_bytes(payload)
    raise IoFailure("no input volume: pass -i PATH or pipe volume bytes")


def _write_bytes_out(path, payload: bytes) -> None:
    """Payload to standard output, or atomically to ``path`` (io.atomic_output)."""
    if path:
        with vio.atomic_output(path) as fh:
            fh.write(payload)
        return
    out = sys.stdout.buffer
    out.write(payload)
    out.flush()


def _write_volume_out(args, volume) -> None:
    _write_bytes_out(getattr(args, "output", None), vio.volume_to_bytes(volume))


def _kernel(args):
    """--gaussian SIGMA [--ksize K], or --kernel-file: whitespace-separated
    tokens, three integer extents then the x-fastest weights (cli.py:363-372)."""
    from .filters import Kernel, gaussian_kernel

    if (args.gaussian is None) == (args.kernel_file is None):
        raise InvalidArgument("pass exactly one of --gaussian or --kernel-file")
    if args.kernel_file is None:
        return gaussian_kernel(args.gaussian, args.ksize)
    try:
        tokens = Path(args.kernel_file).read_text().split()
    except OSError as exc:
        raise IoFailure(str(exc)) from exc
    extents = tuple(int(t) for t in tokens[:3])
    return Kernel(extents, np.array(tokens[3:], dtype=np.float64))


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
    payload = _input_bytes(args)
    volume = vio.load_raw(payload, args.dims, args.format, args.cell_size, tuple(args.range))
    _write_volume_out(args, volume)
    return 0


def _cmd_bench(args) -> int:
    """The structured cases of the reference bench on the B200
    (benchmarks.run_benchmarks; report lines as cli.py:495-509)."""
    from .benchmarks import run_benchmarks

    reports = run_benchmarks(args.size, args.subgrids, args.bench_workers, args.repeat)
    text = "".join(f"bench: case={r['case']} serial_s={r['serial_s']:.6f} "
                   f"parallel_s={r['parallel_s']:.6f} workers={r['workers']} "
                   f"effective_workers={r['effective_workers']}\n" for r in reports)
    _write_bytes_out(getattr(args, "output", None), text.encode())
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


def _error_line(exc: BaseException) -> str:
    """``error: <ErrorName>: <message>`` — the line the TS bindings parse
    (cli.ts:38); OS errors report as IoFailure (cli.py:559-564)."""
    name = exc.name if isinstance(exc, VktError) else "IoFailure"
    return f"error: {name}: {exc}\n"


def main(argv=None) -> int:
    """Exit status 0 on success, 1 on a usage error, 2 on a data error."""
    try:
        args = _build_parser().parse_args(argv)
    except SystemExit as stop:
        return int(stop.code or 0)
    set_execution_policy(ExecutionPolicy(worker_count=args.workers, print_timings=args.timings))
    command = _COMMANDS[args.command]
    try:
        return command(args)
    except (VktError, OSError) as exc:
        sys.stderr.write(_error_line(exc))
        return 2


if __name__ == "__main__":
    sys.exit(main())
