"""Execution policy for the device path.

The reference carries a frozen, thread-local ``ExecutionPolicy`` that selects
the device space and a worker-count bound (pkg/src/vkt/execution.py:37-65) and
runs ``apply_filter`` as ≤64 z-slabs on a thread pool (:113-170).  On the B200
the slab/thread decomposition is replaced by the CUDA grid, so the policy here
selects the CUDA device, the kernel path (tiled TMA kernel, generic direct
kernel, or the bit-exact float64 mode) and the timing printout.  The API shape
(thread-local set/get, ``timed``) is kept so caller code does not change.
"""

from __future__ import annotations

import sys
import threading
import time
from dataclasses import dataclass, replace
from enum import Enum
from functools import wraps


class Device(Enum):
    CUDA = "cuda"


class FilterPath(Enum):
    AUTO = "auto"      # tiled TMA kernel when it applies, else direct
    DIRECT = "direct"  # generic one-output-per-thread kernel
    EXACT = "exact"    # float64, bit-exact with the reference arithmetic


@dataclass(frozen=True)
class ExecutionPolicy:
    """Per-thread settings for subsequent calls.

    ``worker_count`` is accepted for signature compatibility with the
    reference (execution.py:45) and ignored: the device grid decides.
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


def set_execution_policy(policy: ExecutionPolicy) -> None:
    _local.policy = policy


def get_execution_policy() -> ExecutionPolicy:
    return getattr(_local, "policy", _DEFAULT)


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
