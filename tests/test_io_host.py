"""CPU: VKTVOL01 header logic against files written by the reference."""

import struct

import numpy as np
import pytest

import paper_2203_10213_b200 as vk
from paper_2203_10213_b200 import io as vio
from conftest import GOLDEN

FILES = {"u8": vk.DataFormat.UINT8, "u16": vk.DataFormat.UINT16, "f32": vk.DataFormat.FLOAT32}


@pytest.mark.parametrize("short", list(FILES))
def test_header_roundtrip_matches_reference_bytes(short):
    raw = (GOLDEN / f"vol_{short}.vkt").read_bytes()
    dims, fmt, cell, mapping = vio.parse_header(raw[:vio.HEADER_SIZE])
    assert fmt is FILES[short]
    assert len(raw) == vio.HEADER_SIZE + dims.x * dims.y * dims.z * fmt.bytes_per_cell
    assert vio.pack_header(dims, fmt, cell, mapping) == raw[:vio.HEADER_SIZE]
    assert vio.HEADER_SIZE == 42


def test_header_errors_use_reference_names():
    good = (GOLDEN / "vol_u8.vkt").read_bytes()[:vio.HEADER_SIZE]
    with pytest.raises(vk.BadMagic):
        vio.parse_header(b"NOTAVOL!" + good[8:])
    with pytest.raises(vk.TruncatedPayload):
        vio.parse_header(good[:20])
    bad_code = bytearray(good)
    bad_code[21] = 9
    with pytest.raises(vk.UnknownFormatCode):
        vio.parse_header(bytes(bad_code))
    bad_type = bytearray(good)
    bad_type[8] = 7
    with pytest.raises(vk.UnknownFormatCode):
        vio.parse_header(bytes(bad_type))
    hier = bytearray(good)
    hier[8] = 1
    with pytest.raises(vk.InvalidArgument):
        vio.parse_header(bytes(hier))


def test_cli_usage_and_missing_input_exit_codes():
    import subprocess
    import sys

    r = subprocess.run([sys.executable, "-m", "paper_2203_10213_b200", "frobnicate"], capture_output=True)
    assert r.returncode == 1
    r = subprocess.run([sys.executable, "-m", "paper_2203_10213_b200", "info", "-i", "/nonexistent.vkt"],
                       capture_output=True)
    assert r.returncode == 2 and b"error: IoFailure:" in r.stderr
    r = subprocess.run([sys.executable, "-m", "paper_2203_10213_b200", "info", "-i",
                        str(GOLDEN / "vol_u16.vkt")], capture_output=True)
    assert r.returncode == 0
    text = r.stdout.decode()
    assert "16x8x11" in text and "u16" in text and "range: -1 3" in text
