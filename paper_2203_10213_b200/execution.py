"""Execution policy for the device path.

The reference carries a frozen, thread-local ``ExecutionPolicy`` that selects
the device space and a worker-count bound (pkg/src/vkt/execution.py:37-65) and
runs ``apply_filter`` as ≤64 z-slabs on a thread pool (:113-170).  On the B200
the slab/thread decomposition is replaced by the CUDA grid, so the policy here
selects where a ``ManagedBuffer`` lives, the CUDA device, the kernel path
(tiled TMA kernel, generic direct kernel, or the bit-exact float64 mode) and
the timing printout.  The API shape (thread-local set/get, ``timed``,
``effective_workers``) is kept so caller code does not change.

Device spaces (``ExecutionPolicy.device``):
  * ``Device.CPU`` — the reference's default: volume bytes in page-locked
    host memory, ``array()`` is a writable numpy view.  Every algorithm still
    computes on the B200 (ApplyFilter streams the host buffer through HBM,
    Fill stores into the mapped host buffer); there is no CPU compute path.
  * ``Device.EMULATED_DEVICE`` — the reference's stand-in for an accelerator
    (managed.py:31-59); here it IS the accelerator: bytes in HBM.
  * ``Device.CUDA`` — HBM residency under this package's own name.
"""

from __future__ import annotations

import os
import sys
import threading
import time
from dataclasses import dataclass, replace
from enum import Enum
from functools import wraps


class Device(Enum):
    CPU = "cpu"                   # host residency (reference default, execution.py:32-34)
    EMULATED_DEVICE = "emulated"  # HBM (the reference's emulated accelerator)
    CUDA = "cuda"                 # HBM

    @property
    def on_host(self) -> bool:
        return self is Device.CPU


class FilterPath(Enum):
    AUTO = "auto"      # separable kernel for rank-1 weights, else dense tiled, else direct
    DENSE = "dense"    # as AUTO without the separable kernel (bit-identical to DIRECT)
    DIRECT = "direct"  # generic one-output-per-thread kernel
    EXACT = "exact"    # float64, bit-exact with the reference arithmetic


@dataclass(frozen=True)
class ExecutionPolicy:
    """Per-thread settings for subsequent calls.

    ``worker_count`` bounds host threads exactly like the reference's
    (execution.py:40-48, ``effective_workers``); the device grid does not
    depend on it, so results never do either.  ``device`` picks the residency
    of ``ManagedBuffer`` volumes (module docstring); the native API's
    ``DeviceBuffer`` volumes always live in HBM.
    """

    device: Device = Device.CUDA
    device_index: int | None = None
    worker_count: int = 0
    print_timings: bool = False
    debug_messages: bool = False
    filter_path: FilterPath = FilterPath.AUTO

    def __post_init__(self) -> None:
        if self.worker_count < 0:
            raise ValueError("worker_count must be >= 0")
        if not isinstance(self.filter_path, FilterPath):
            object.__setattr__(self, "filter_path", FilterPath(self.filter_path))


_local = threading.local()
_DEFAULT = ExecutionPolicy()


_hw_override: int | None = None


def set_hardware_concurrency_override(n: int | None) -> None:
    """Pretend ``n`` host threads are available, None restores the real count
    (execution.py:71-82).  Device results are unaffected either way."""
    global _hw_override
    if n is not None and n < 1:
        raise ValueError("hardware concurrency must be >= 1")
    _hw_override = n


def hardware_concurrency() -> int:
    """Host threads this process may run on (execution.py:84-89)."""
    if _hw_override is not None:
        return _hw_override
    try:
        return len(os.sched_getaffinity(0))
    except AttributeError:
        return os.cpu_count() or 1


def effective_workers(policy: "ExecutionPolicy | None" = None) -> int:
    """Host threads a call runs with under ``policy`` (execution.py:92-97):
    the requested count (0 = all) clamped to ``hardware_concurrency()``."""
    policy = policy or get_execution_policy()
    hw = hardware_concurrency()
    return max(1, min(policy.worker_count or hw, hw))


def set_execution_policy(policy: ExecutionPolicy) -> None:
    _local.policy = policy


def get_execution_policy() -> ExecutionPolicy:
    return getattr(_local, "policy", _DEFAULT)


def explicit_policy() -> "ExecutionPolicy | None":
    """The policy set on this thread, or None when none was set (managed
    buffers then follow the reference's default, host residency)."""
    return getattr(_local, "policy", None)


def with_policy(**changes) -> ExecutionPolicy:
    return replace(get_execution_policy(), **changes)


def debug(msg: str) -> None:
    if get_execution_policy().debug_messages:
        print(f"[vkt] {msg}", file=sys.stderr)


def timed(name: str):
    """Print the wall time of the call (device work included) when asked.

    Same output line as the reference (execution.py:178-196); the device is
    synchronized before reading the clock so the number covers the kernels.
    """

    def deco(fn):
        @wraps(fn)
        def wrapper(*args, **kwargs):
            if not get_execution_policy().print_timings:
                return fn(*args, **kwargs)
            import torch

            torch.cuda.synchronize()
            t0 = time.perf_counter()
            try:
                return fn(*args, **kwargs)
            finally:
                torch.cuda.synchronize()
                print(f"[vkt] {name}: {time.perf_counter() - t0:.6f} s", file=sys.stderr)

        return wrapper

    return deco
