"""CPU: the reference-compatible namespace (paper_2203_10213_b200.vkt) and the
host-side pieces of the drop-in that need no GPU."""

import os
import stat

import pytest

import paper_2203_10213_b200 as vk
import paper_2203_10213_b200.vkt as vkt
from paper_2203_10213_b200 import io as vio


def test_policy_defaults_follow_the_reference():
    # execution.py:37-51: the reference's default device is the CPU (host residency)
    assert vkt.ExecutionPolicy().device is vkt.Device.CPU
    assert vk.ExecutionPolicy().device is vk.Device.CUDA
    assert vkt.Device.EMULATED_DEVICE.value == "emulated" and vkt.Device.CPU.on_host
    vkt.set_execution_policy(vkt.ExecutionPolicy(worker_count=3))
    try:
        assert vkt.get_execution_policy().worker_count == 3
        assert vk.get_execution_policy() is vkt.get_execution_policy()
    finally:
        vkt.set_execution_policy(vkt.ExecutionPolicy())
    with pytest.raises(ValueError):
        vkt.ExecutionPolicy(worker_count=-1)


def test_effective_workers_and_override():
    # execution.py:71-97
    vkt.set_hardware_concurrency_override(8)
    try:
        assert vkt.hardware_concurrency() == 8
        assert vkt.effective_workers(vkt.ExecutionPolicy(worker_count=1)) == 1
        assert vkt.effective_workers(vkt.ExecutionPolicy(worker_count=64)) == 8
        assert vkt.effective_workers(vkt.ExecutionPolicy()) == 8
    finally:
        vkt.set_hardware_concurrency_override(None)
    assert vkt.hardware_concurrency() == len(os.sched_getaffinity(0))
    with pytest.raises(ValueError):
        vkt.set_hardware_concurrency_override(0)


def test_device_space_capacity_accounting():
    space = vk.volume.DeviceSpace()
    space.set_capacity(100)
    space.reserve(60)
    with pytest.raises(vk.AllocationFailure):
        space.reserve(50)
    space.release(60)
    space.reserve(100)
    assert vkt.emulated_device.capacity_bytes is None


def test_reference_error_names_and_modules():
    from paper_2203_10213_b200.vkt import errors as E
    from paper_2203_10213_b200.vkt.ops.filters import _clip_counts, brick_mappings  # noqa: F401

    for name in ("InvalidArgument", "EvenKernelDims", "AllocationFailure", "DimsMismatch",
                 "EmptyRange", "NotASlab", "RangeOutOfBounds", "IndexOutOfRange"):
        cls = getattr(E, name)
        assert issubclass(cls, vkt.VktError) and cls("x").name == name
    with pytest.raises(E.EvenKernelDims):
        vkt.Kernel((2, 3, 3), [0.0] * 18)
    assert vkt.StructuredVolume._new_storage.__func__ is not vk.StructuredVolume._new_storage.__func__


def test_atomic_output_mode_and_no_partial(tmp_path):
    target = tmp_path / "out.bin"
    with vio.atomic_output(target) as fh:
        fh.write(b"abc")
    assert target.read_bytes() == b"abc"
    mask = os.umask(0)
    os.umask(mask)
    assert stat.S_IMODE(target.stat().st_mode) == 0o666 & ~mask
    os.chmod(target, 0o640)
    with pytest.raises(RuntimeError):
        with vio.atomic_output(target) as fh:
            fh.write(b"partial")
            raise RuntimeError("boom")
    assert target.read_bytes() == b"abc"
    assert [p.name for p in tmp_path.iterdir()] == ["out.bin"]
    with vio.atomic_output(target) as fh:
        fh.write(b"new")
    assert stat.S_IMODE(target.stat().st_mode) == 0o640  # existing mode kept


def test_cli_usage_error_exit_1(capsys):
    from paper_2203_10213_b200 import cli

    assert cli.main(["filter", "--bogus"]) == 1
    err = capsys.readouterr().err
    assert "usage:" in err and "error: unrecognized arguments: --bogus" in err


def test_cli_error_line_format():
    from paper_2203_10213_b200 import cli

    assert cli._error_line(vk.InvalidArgument("bad")) == "error: InvalidArgument: bad\n"
    assert cli._error_line(FileNotFoundError(2, "No such file")).startswith("error: IoFailure: ")


def test_with_policy_uses_the_reference_default():
    p = vkt.with_policy(worker_count=5)
    assert p.device is vkt.Device.CPU and p.worker_count == 5
    assert vkt.get_execution_policy().worker_count == 0  # not installed
