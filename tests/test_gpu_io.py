"""GPU: VKTVOL01 I/O into HBM, range I/O, out-of-core filter_file and the CLI,
against files and CLI outputs produced by the reference (oracle/make_golden.py)."""

import subprocess
import sys

import numpy as np
import pytest

import paper_2203_10213_b200 as vk
from paper_2203_10213_b200 import io as vio
from conftest import GOLDEN, within_contract
from oracle import vkt_oracle as O

pytestmark = pytest.mark.gpu
CLI = [sys.executable, "-m", "paper_2203_10213_b200"]
SHORTS = ["u8", "u16", "f32"]


def _payload(path):
    raw = path.read_bytes()
    dims, fmt, _, _ = vio.parse_header(raw[:vio.HEADER_SIZE])
    return np.frombuffer(raw[vio.HEADER_SIZE:], dtype=fmt.dtype).reshape(dims.z, dims.y, dims.x), fmt


@pytest.mark.parametrize("short", SHORTS)
def test_read_write_roundtrip_bit_exact(short, tmp_path):
    path = GOLDEN / f"vol_{short}.vkt"
    v = vk.read_volume(path)
    host, fmt = _payload(path)
    assert np.array_equal(v.to_numpy(), host)
    out = tmp_path / "o.vkt"
    vk.write_volume(out, v)
    assert out.read_bytes() == path.read_bytes()
    assert vk.volume_to_bytes(vk.volume_from_bytes(path.read_bytes())) == path.read_bytes()


@pytest.mark.parametrize("short", SHORTS)
def test_range_io(short, tmp_path):
    path = GOLDEN / f"vol_{short}.vkt"
    host, fmt = _payload(path)
    nz, ny, nx = host.shape
    for lo, hi in (((0, 0, 2), (nx, ny, 5)), ((0, 3, 1), (nx, ny - 1, 4)), ((2, 1, 0), (7, 6, 3))):
        r = vk.read_range(path, (lo, hi))
        assert np.array_equal(r.to_numpy(), host[lo[2]:hi[2], lo[1]:hi[1], lo[0]:hi[0]])
    with pytest.raises(vk.RangeOutOfBounds):
        vk.read_range(path, ((0, 0, 0), (nx + 1, ny, nz)))
    with pytest.raises(vk.EmptyRange):
        vk.read_range(path, ((1, 1, 1), (1, 2, 2)))
    target = tmp_path / "t.vkt"
    target.write_bytes(path.read_bytes())
    sub = vk.StructuredVolume.from_numpy(np.zeros((2, 3, 4), dtype=fmt.dtype), fmt)
    vk.write_range(target, sub, (1, 2, 3))
    got, _ = _payload(target)
    want = host.copy()
    want[3:5, 2:5, 1:5] = 0
    assert np.array_equal(got, want)


@pytest.mark.parametrize("mode", ["clamp", "wrap", "mirror", "border"])
@pytest.mark.parametrize("short,k,chunk", [("u16", 7, 3), ("f32", 3, 1), ("u8", 5, 4)])
def test_filter_file_out_of_core_matches_device(mode, short, k, chunk, tmp_path):
    path = GOLDEN / f"vol_{short}.vkt"
    kern = vk.gaussian_kernel(1.0, k) if k != 5 else vk.box_kernel(5)
    out = tmp_path / "f.vkt"
    vk.filter_file(path, out, kern, mode, chunk_planes=chunk)
    v = vk.read_volume(path)
    dst = vk.StructuredVolume(v.dims, v.format, v.cell_size, v.mapping)
    vk.ApplyFilter(dst, v, kern, mode)
    assert out.read_bytes() == vk.volume_to_bytes(dst)


@pytest.mark.parametrize("short", SHORTS)
def test_cli_filter_matches_reference_cli(short, tmp_path):
    """`filter --gaussian 1.0 --ksize 3` on the reference's files vs the
    reference CLI's own output files: same header, payload within contract."""
    src = GOLDEN / f"vol_{short}.vkt"
    ref_out = GOLDEN / f"filtered_vol_{short}.vkt"
    ours = tmp_path / "o.vkt"
    r = subprocess.run(CLI + ["filter", "--gaussian", "1.0", "--ksize", "3", "-i", str(src), "-o", str(ours)],
                       capture_output=True, timeout=300)
    assert r.returncode == 0, r.stderr
    got_raw, want_raw = ours.read_bytes(), ref_out.read_bytes()
    assert got_raw[:vio.HEADER_SIZE] == want_raw[:vio.HEADER_SIZE]
    got, fmt = _payload(ours)
    want, _ = _payload(ref_out)
    ok, ndiff, dmax = within_contract(got, want, fmt.value, vk.gaussian_kernel(1.0, 3).weights)
    assert ok, (ndiff, dmax)
    # pipes: stdin -> stdout
    r = subprocess.run(CLI + ["filter", "--gaussian", "1.0", "--ksize", "3"], input=src.read_bytes(),
                       capture_output=True, timeout=300)
    assert r.returncode == 0 and r.stdout == got_raw


def test_cli_fill_kernel_file_timings_and_no_partial_output(tmp_path):
    src = GOLDEN / "vol_u8.vkt"
    host, fmt = _payload(src)
    o = tmp_path / "fill.vkt"
    r = subprocess.run(CLI + ["--timings", "fill", "--value", "0.5", "--roi", "1", "1", "1", "5", "5", "5",
                              "-i", str(src), "-o", str(o)], capture_output=True, timeout=300)
    assert r.returncode == 0 and b"FillRange" in r.stderr
    got, _ = _payload(o)
    assert np.array_equal(got, O.fill_range(host, 1, (1, 1, 1), (5, 5, 5), 0.5))
    # kernel file: forward-x shift (pkg/tests/test_ops_filter.py:50-57)
    kf = tmp_path / "k.txt"
    kf.write_text("3 1 1\n0 0 1\n")
    o2 = tmp_path / "shift.vkt"
    r = subprocess.run(CLI + ["filter", "--kernel-file", str(kf), "--mode", "wrap", "-i", str(src), "-o", str(o2)],
                       capture_output=True, timeout=300)
    assert r.returncode == 0, r.stderr
    got, _ = _payload(o2)
    assert np.array_equal(got, np.roll(host, -1, axis=2))
    # a failing invocation leaves the existing output untouched
    target = tmp_path / "precious.vkt"
    target.write_bytes(b"precious")
    r = subprocess.run(CLI + ["filter", "--gaussian", "1.0", "--ksize", "4", "-i", str(src), "-o", str(target)],
                       capture_output=True, timeout=300)
    assert r.returncode == 2 and b"error: EvenKernelDims:" in r.stderr
    assert target.read_bytes() == b"precious"


def test_cli_bench_shape():
    r = subprocess.run(CLI + ["bench", "--size", "64", "--repeat", "2"], capture_output=True, timeout=300)
    assert r.returncode == 0, r.stderr
    rows = {}
    for line in r.stdout.decode().strip().splitlines():
        fields = dict(kv.split("=") for kv in line.split()[1:])
        rows[fields["case"]] = fields
    g = rows["gaussian_filter"]
    assert float(g["parallel_s"]) <= float(g["serial_s"])
