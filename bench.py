#!/usr/bin/env python
"""ApplyFilter benchmark (BASELINE.json metric) — one JSON line on rank 0.

Workloads (``--config``):
  cfg3 (default, BASELINE.json configs[2]): 7x7x7 Gaussian (gaussian_kernel(1.5),
       SURVEY §8(d)) on a 1024^3 uint16 volume, Clamp (the reference's only
       mode), z-slab sharded with NCCL halo exchange at N = 1/2/4/8 GPUs;
  cfg4 (BASELINE.json configs[3]): the 7-point Laplacian in a 3^3 footprint on
       a 2048^3 float32 volume (32 GiB), Wrap, z-slab sharded.
Both scale strongly (the volume is fixed).  A "step" is one ApplyFilter pass
over the whole volume, on the default path: the Gaussian is rank-1, so cfg3
runs the separable kernel (csrc/filter_sep.cuh); ``dense_kernel`` in the line
times the same workload on the dense tiled kernel (filter_path="dense").

  python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference] [--config cfg3|cfg4]

With --gpus N > 1 and no WORLD_SIZE in the environment the script launches
itself under torch.distributed.run (one process per GPU, 127.0.0.1); the
torchrun form works as well:
  python -m torch.distributed.run --nnodes=1 --nproc-per-node N \\
      --master-addr 127.0.0.1 --master-port P bench.py --gpus N ...
NCCL's INIT lines (NCCL_DEBUG=INFO, NCCL_DEBUG_SUBSYS=INIT) go to stderr.

Timing: W untimed warm-up steps; K timed steps bracketed by a barrier and
cuda synchronize; CUDA events on the launching stream; max over ranks.  Both
inputs are larger than the 126 MB L2 (2.1 GB / 34 GB; >= 268 MB per rank at
N = 8), so no flush is needed between steps.

--impl reference (and the ``cpu_baseline`` leg of ours, rank 0 at N = 1) time
the reference's own CPU implementation of the path, ``vkt.apply_filter``
(pkg/src/vkt/ops/filters.py:69-95, the unmodified package installed in
baseline/_ref; the oracle port oracle/vkt_oracle.py when that is absent), on
all host threads, over a sample of the workload: full-width rows, 4 planes
per host thread (the reference cuts z into 4-plane slabs at this depth,
execution.py:162-170, so every thread gets one slab), as many rows (up to the
full plane) as the time budget allows.  Full planes keep each numpy pass
DRAM-sized like the full-volume run's; profiles/r02_cpu_baseline_sweep.txt
records the rate against the sample shape.
"""

from __future__ import annotations

import argparse
import json
import os
import socket
import statistics
import subprocess
import sys
import time
from pathlib import Path

ROOT = Path(__file__).resolve().parent
sys.path.insert(0, str(ROOT))

METRIC = "ApplyFilter GVoxels/s at 1/2/4/8 B200; % of HBM/FP32 roofline"
UNIT = "GVox/s"
CONFIGS = {
    "cfg3": dict(workload="cfg3: ApplyFilter 7x7x7 Gaussian(sigma=1.5) on 1024^3 uint16, Clamp, "
                          "z-slab sharded with NCCL halo exchange",
                 dims=[1024, 1024, 1024], format="u16", kernel="gaussian_kernel(1.5) 7x7x7",
                 address_mode="clamp"),
    "cfg4": dict(workload="cfg4: ApplyFilter 3x3x3 7-point Laplacian on 2048^3 float32 (32 GiB), Wrap, "
                          "z-slab sharded with NCCL halo exchange",
                 dims=[2048, 2048, 2048], format="f32", kernel="laplacian 3x3x3 (centre -6, faces +1)",
                 address_mode="wrap"),
}
NCCL_ENV = {"NCCL_DEBUG": "INFO", "NCCL_DEBUG_SUBSYS": "INIT", "NCCL_DEBUG_FILE": "/dev/stderr"}


def workload(name):
    import paper_2203_10213_b200 as vk

    if name == "cfg4":
        return CONFIGS[name], vk.DataFormat.FLOAT32, vk.laplacian_kernel(), vk.AddressMode.WRAP
    return CONFIGS[name], vk.DataFormat.UINT16, vk.gaussian_kernel(1.5), vk.AddressMode.CLAMP


def config_dict(name, n):
    """Identical in both arms (the reference arm describes its execution in
    cpu_baseline.sample)."""
    return dict(CONFIGS[name], parallelism=f"z-slab x{n}")


def load_peaks():
    p = ROOT / "MEASURED_PEAKS.json"
    if p.exists():
        d = json.loads(p.read_text())
        return float(d.get("hbm_gbs", 6650.0)), float(d.get("sm_max_mhz", 1965.0)), "measured"
    return 6650.0, 1965.0, "fallback"


class ClockSampler:
    """nvidia-smi clocks + throttle reasons sampled during the timed region."""

    FIELDS = ("clocks.sm,clocks.max.sm,clocks_event_reasons.hw_slowdown,"
              "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
              "clocks_event_reasons.sw_power_cap")

    def __init__(self, index: int):
        self.index = index
        self.proc = None

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.FIELDS}",
                 "--format=csv,noheader,nounits", "-lms", "100"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
        except OSError:
            self.proc = None
        return self

    def __exit__(self, *exc):
        self.lines = []
        if self.proc is not None:
            time.sleep(0.15)
            self.proc.terminate()
            try:
                out, _ = self.proc.communicate(timeout=5)
            except subprocess.TimeoutExpired:
                self.proc.kill()
                out, _ = self.proc.communicate()
            self.lines = [l for l in out.splitlines() if l.strip()]

    def summary(self):
        names = ("hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap")
        sm, mx, reasons = [], [], set()
        for line in getattr(self, "lines", []):
            parts = [p.strip() for p in line.split(",")]
            if len(parts) < 6:
                continue
            try:
                sm.append(float(parts[0]))
                mx.append(float(parts[1]))
            except ValueError:
                continue
            for n, v in zip(names, parts[2:6]):
                if v.lower().startswith("active"):
                    reasons.add(n)
        return {"sm_mhz": statistics.median(sm) if sm else None,
                "sm_max_mhz": max(mx) if mx else None,
                "reasons": sorted(reasons), "samples": len(sm)}


def _free_port() -> int:
    with socket.socket(socket.AF_INET, socket.SOCK_STREAM) as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def spawn_ranks(n: int) -> int:
    """Re-run this script as N ranks under torch.distributed.run (one process
    per GPU); rank 0's JSON line comes through on stdout."""
    env = dict(os.environ)
    for k, v in NCCL_ENV.items():
        env.setdefault(k, v)
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={n}",
           "--master-addr", "127.0.0.1", "--master-port", str(_free_port()), str(Path(__file__).resolve()),
           *sys.argv[1:]]
    return subprocess.run(cmd, env=env).returncode


def dist_setup(n_gpus: int, test_single_gpu: bool = False):
    """One process per GPU over NCCL.  ``test_single_gpu`` (testing only) runs
    all ranks on cuda:0 over gloo with host-staged halo exchange, because
    NCCL's spinning P2P kernels must not share one device."""
    import torch
    import torch.distributed as dist

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = 0 if test_single_gpu else int(os.environ.get("LOCAL_RANK", "0"))
    if world != n_gpus:
        raise SystemExit(f"--gpus {n_gpus} but WORLD_SIZE={world}")
    torch.cuda.set_device(local)
    if world > 1:
        os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
        for k, v in NCCL_ENV.items():
            os.environ.setdefault(k, v)
        if test_single_gpu:
            dist.init_process_group("gloo")
        else:
            dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    return rank, world, local


# ---------------------------------------------------------------------------
# CPU reference (the reference's own apply_filter on the host cores)
# ---------------------------------------------------------------------------

def _reference_vkt():
    """The unmodified reference package from baseline/_ref, or None."""
    ref = ROOT / "baseline" / "_ref"
    if not (ref / "vkt" / "__init__.py").exists():
        return None
    if str(ref) not in sys.path:
        sys.path.insert(0, str(ref))
    try:
        import vkt  # noqa: F401  (the reference, not this package)
    except Exception:
        return None
    return sys.modules["vkt"]


def cpu_reference(cfg_name: str, budget_s: float, steps: int, warmup: int):
    """Time the reference apply_filter on a sample of the workload.

    Sample: 1024 (cfg3) / 2048 (cfg4) cells per row, ``4 * threads`` planes
    (one 4-plane reference slab per host thread), rows chosen so one step
    takes about ``budget_s``.  Returns (GVox/s over the timed steps, info)."""
    import numpy as np

    threads = len(os.sched_getaffinity(0))
    nx = CONFIGS[cfg_name]["dims"][0]
    planes = 4 * threads
    vkt = _reference_vkt()
    rng = np.random.default_rng(7)
    is_f32 = cfg_name == "cfg4"

    if vkt is not None:
        vkt.set_execution_policy(vkt.ExecutionPolicy(worker_count=0))
        fmt = vkt.DataFormat.FLOAT32 if is_f32 else vkt.DataFormat.UINT16
        if is_f32:
            w = np.zeros((3, 3, 3))
            w[1, 1, 1] = -6.0
            for z, y, x in ((0, 1, 1), (2, 1, 1), (1, 0, 1), (1, 2, 1), (1, 1, 0), (1, 1, 2)):
                w[z, y, x] = 1.0
            kern = vkt.Kernel((3, 3, 3), w.reshape(-1))
        else:
            kern = vkt.gaussian_kernel(1.5)

        def make(rows):
            v = vkt.StructuredVolume((nx, rows, planes), fmt)
            a = v.array()
            a[...] = (rng.random(a.shape, dtype=np.float32) if is_f32
                      else rng.integers(0, 65536, size=a.shape, dtype=np.uint16))
            return v

        def run(v):
            t0 = time.perf_counter()
            vkt.apply_filter(v, kern)  # in place; the next call filters the result, same cost
            return time.perf_counter() - t0

        kind, workers = "reference", vkt.effective_workers()
        impl = "vkt.apply_filter (baseline/_ref, unmodified reference, filters.py:69-95)"
    else:
        from oracle import vkt_oracle as O

        w = O.laplacian_weights() if is_f32 else O.gaussian_weights(1.5)

        def make(rows):
            return (rng.random((planes, rows, nx), dtype=np.float32) if is_f32
                    else rng.integers(0, 65536, size=(planes, rows, nx), dtype=np.uint16))

        def run(v):
            t0 = time.perf_counter()
            O.apply_filter(v, 3 if is_f32 else 2, w, "clamp", workers=threads)
            return time.perf_counter() - t0

        kind, workers = "port", threads
        impl = "oracle/vkt_oracle.py apply_filter (port of filters.py:69-95)"

    probe_rows = 256
    t_probe = run(make(probe_rows))  # calibration, untimed
    per_row = t_probe / probe_rows
    # >= 512 rows keeps every numpy pass >= 16 MB (DRAM-sized, like the full run's)
    rows = int(max(512, min(CONFIGS[cfg_name]["dims"][1], budget_s / max(per_row, 1e-6))))
    vol = make(rows)
    times = []
    for i in range(warmup + steps):
        dt = run(vol)
        if i >= warmup:
            times.append(dt)
    total = sum(times)
    nvox = nx * rows * planes
    value = nvox * len(times) / total / 1e9
    info = dict(cores=workers, kind=kind, seconds=total, rows=rows, planes=planes,
                sample=(f"{impl}: {nx}x{rows}x{planes} {'f32' if is_f32 else 'u16'} volume "
                        f"({planes // 4} slabs of 4 planes = 1 per host thread), "
                        f"{'laplacian 3^3' if is_f32 else 'gaussian 7^3'}, Clamp (the reference's "
                        f"only mode; same tap-loop cost as Wrap), {len(times)} timed step(s)"))
    return value, info


def run_reference(args):
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    steps, warmup = args.steps, args.warmup
    budget = max(0.25, min(args.cpu_budget, 200.0 / max(1, steps + warmup)))
    value, info = cpu_reference(args.config, budget, steps, warmup)
    ms = info["seconds"] / max(1, steps) * 1e3
    line = {
        "metric": METRIC, "value": round(value, 6), "unit": UNIT, "impl": "reference",
        "n_gpus": args.gpus, "steps": steps, "warmup": warmup, "ms_per_step": round(ms, 3),
        "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "f64",
        "data": "synthetic (numpy default_rng(7), the reference generator's distribution)",
        "config": config_dict(args.config, args.gpus),
        "cpu_baseline": {"value": round(value, 6), "unit": UNIT, "cores": info["cores"],
                         "kind": info["kind"], "sample": info["sample"]},
        "e2e": {"value": round(value, 6), "unit": UNIT, "h2d_bytes_per_step": 0,
                "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


# ---------------------------------------------------------------------------
# Our arm
# ---------------------------------------------------------------------------

def algorithmic_fma(kernel, path):
    """FMAs per voxel of the algorithm the path runs: the dense correlation
    evaluates every tap (kx*ky*kz); the separable kernel three 1-D sums
    (kx + ky + kz, csrc/filter_sep.cuh)."""
    kx, ky, kz = kernel.dims
    return kx + ky + kz if path == "separable" else kx * ky * kz


def kernel_rate(weights_kernel, dims=(1024, 1024, 1024), reps=10, fmt=None, path="auto", mode="clamp"):
    """ApplyFilter kernel time on a resident volume (events, median of reps)."""
    import torch

    import paper_2203_10213_b200 as vk

    fmt = fmt or vk.DataFormat.FLOAT32
    vk.set_execution_policy(vk.ExecutionPolicy(filter_path=path))
    try:
        return _kernel_rate(vk, torch, weights_kernel, dims, reps, fmt, mode)
    finally:
        vk.set_execution_policy(vk.ExecutionPolicy())


def _kernel_rate(vk, torch, weights_kernel, dims, reps, fmt, mode):
    src = vk.synthetic_device(dims, fmt, seed=11)
    dst = vk.StructuredVolume(src.dims, src.format, data=vk.DeviceBuffer(src.nbytes, zero=False))
    s = torch.cuda.current_stream()
    for _ in range(2):
        vk.ApplyFilter(dst, src, weights_kernel, mode)
    times = []
    for _ in range(reps):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(s)
        vk.ApplyFilter(dst, src, weights_kernel, mode)
        e1.record(s)
        e1.synchronize()
        times.append(e0.elapsed_time(e1))
    ms = statistics.median(times)
    nvox = dims[0] * dims[1] * dims[2]
    path = vk.filter_path(dst, src, weights_kernel, mode)
    del src, dst
    torch.cuda.empty_cache()
    return ms, nvox, path


def roofline_obj(nvox, ms, bpc, taps, hbm_gbs, sm_mhz_max, nsm):
    """Slower of HBM (2*bpc bytes/voxel) and FP32 (taps FMAs/voxel) bounds."""
    fma_peak = nsm * 128 * sm_mhz_max * 1e6  # FMA/s
    t_hbm = nvox * 2 * bpc / (hbm_gbs * 1e9)
    t_fma = nvox * taps / fma_peak
    sec = ms / 1e3
    if t_fma >= t_hbm:
        achieved = nvox * taps * 2 / sec / 1e12
        return {"bound": "fp32", "achieved": round(achieved, 3), "peak": round(fma_peak * 2 / 1e12, 3),
                "unit": "TFLOP/s", "frac": round(achieved / (fma_peak * 2 / 1e12), 4)}
    achieved = nvox * 2 * bpc / sec / 1e9
    return {"bound": "hbm", "achieved": round(achieved, 1), "peak": hbm_gbs, "unit": "GB/s",
            "frac": round(achieved / hbm_gbs, 4)}


def run_ours(args):
    import numpy as np
    import torch
    import torch.distributed as dist

    import paper_2203_10213_b200 as vk
    from paper_2203_10213_b200 import _capi
    from paper_2203_10213_b200.shard import ShardedVolume, apply_filter_sharded

    rank, world, local = dist_setup(args.gpus, args.test_single_gpu)
    dev = torch.device("cuda", local)
    wl, fmt, kernel, mode = workload(args.config)
    nx, ny, nz = wl["dims"]
    src = ShardedVolume((nx, ny, nz), fmt, rank, world, device=dev)
    dst = ShardedVolume((nx, ny, nz), fmt, rank, world, device=dev)
    gen = vk.synthetic_device((nx, ny, nz), fmt, seed=7, z_offset=src.z0, local_nz=src.z1 - src.z0,
                              device=dev)
    src.local.swap_storage(gen)
    del gen
    stream = torch.cuda.current_stream(dev)
    group = dist.group.WORLD if world > 1 else None
    exchange = None
    if args.test_single_gpu and world > 1:
        from paper_2203_10213_b200.shard import exchange_halos_host_staged

        exchange = lambda *a: exchange_halos_host_staged(*a, group=group)  # noqa: E731

    red_dev = torch.device("cpu") if args.test_single_gpu else dev  # gloo reduces on the host

    def allreduce(vals, op):
        t = torch.tensor(vals, device=red_dev, dtype=torch.float64)
        if world > 1:
            dist.all_reduce(t, op=op)
        return [float(v) for v in t.cpu()]

    def allgather(vals):
        t = torch.tensor(vals, device=red_dev, dtype=torch.float64)
        if world == 1:
            return [[float(v) for v in t.cpu()]]
        out = [torch.empty_like(t) for _ in range(world)]
        dist.all_gather(out, t)
        return [[float(v) for v in o.cpu()] for o in out]

    def barrier():
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize(dev)

    barrier()  # every rank's communicator is up before the first P2P batch
    for _ in range(args.warmup):
        apply_filter_sharded(dst, src, kernel, mode, group=group, exchange=exchange)
    barrier()

    launches0 = _capi.launch_count()
    kev: list = []
    phases: dict = {}
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with ClockSampler(local) as clk:
        barrier()
        e0.record(stream)
        for _ in range(args.steps):
            apply_filter_sharded(dst, src, kernel, mode, group=group, exchange=exchange,
                                 kernel_events=kev, phase_events=phases)
        e1.record(stream)
        barrier()
    launches = _capi.launch_count() - launches0
    ms_rank = e0.elapsed_time(e1)
    kern_ms_rank = statistics.mean(a.elapsed_time(b) for a, b in kev)
    exch_ms_rank = statistics.mean(a.elapsed_time(b) for a, b in phases["exchange"]) if phases.get("exchange") else 0.0
    bnd_ms_rank = statistics.mean(a.elapsed_time(b) for a, b in phases["boundary"]) if phases.get("boundary") else 0.0
    per_rank = allgather([ms_rank / args.steps, kern_ms_rank, exch_ms_rank, bnd_ms_rank])
    ms_total, kern_ms = allreduce([ms_rank, kern_ms_rank], dist.ReduceOp.MAX)
    ms_step = ms_total / args.steps
    nvox = nx * ny * nz
    value = nvox / (ms_step / 1e3) / 1e9

    # ---- e2e through the public API with host buffers (pinned) ----
    # vkt_apply_filter_host (paper_2203_10213_b200.apply_filter_host): each
    # rank passes its halo-extended z-slab of the host volume (what range I/O
    # would read); the library streams z-chunks H2D -> filter -> D2H with the
    # three phases overlapped.  Every step moves the slab + halos in and the
    # slab out.  (cfg4 at N = 1 holds 2 x 34 GB of pinned host memory.)
    e2e = None
    if not args.no_e2e:
        e2e_steps = max(1, min(args.steps, args.e2e_steps))
        rz = kernel.radius.z
        plane_b = nx * ny * fmt.bytes_per_cell
        g_planes = [(src.z0 - rz + t) for t in range(rz)] + list(range(src.z0, src.z1)) + \
                   [(src.z1 + t) for t in range(rz)]
        n_in = len(g_planes)
        pin_in = torch.empty(n_in * plane_b, dtype=torch.uint8, pin_memory=True)
        pin_out = torch.empty(n_in * plane_b, dtype=torch.uint8, pin_memory=True)
        from paper_2203_10213_b200.shard import map_plane

        for i, g in enumerate(g_planes):  # halo planes address-mapped (Wrap crosses the faces)
            m = map_plane(g, nz, mode)
            seg = pin_in[i * plane_b:(i + 1) * plane_b]
            if m is None:
                seg.zero_()
            elif src.z0 <= m < src.z1:
                seg.copy_(src.planes()[m - src.z0])
            else:
                h = vk.synthetic_device((nx, ny, nz), fmt, seed=7, z_offset=m, local_nz=1, device=dev)
                seg.copy_(h.data.array)
        host_in = pin_in.numpy().view(fmt.dtype).reshape(n_in, ny, nx)
        host_out = pin_out.numpy().view(fmt.dtype).reshape(n_in, ny, nx)
        zoff = src.z0 - rz  # the buffer's first plane, address-mapped already: pass it as halos
        hl, hh = (host_in[:rz], host_in[n_in - rz:]) if rz else (None, None)
        core_in = host_in[rz:n_in - rz]
        core_out = host_out[rz:n_in - rz]

        def e2e_call():
            vk.apply_filter_host(core_in, kernel, mode, out=core_out, z_offset=src.z0, global_nz=nz,
                                 halo_lo=np.ascontiguousarray(hl) if rz else None,
                                 halo_hi=np.ascontiguousarray(hh) if rz else None)

        del zoff
        for _ in range(max(2, min(args.warmup, 4))):  # grows the library's pools, settles the host side
            e2e_call()
        torch.cuda.synchronize()
        barrier()
        f0, f1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        f0.record(stream)
        for _ in range(e2e_steps):
            e2e_call()
        f1.record(stream)
        barrier()
        e2e_ms = allreduce([f0.elapsed_time(f1)], dist.ReduceOp.MAX)[0] / e2e_steps
        e2e_ok = bool(torch.equal(pin_out[rz * plane_b:(n_in - rz) * plane_b], dst.local.data.array.cpu()))
        h2d_total, d2h_total = (int(v) for v in allreduce([n_in * plane_b, (src.z1 - src.z0) * plane_b],
                                                          dist.ReduceOp.SUM))
        e2e_ok = bool(allreduce([1.0 if e2e_ok else 0.0], dist.ReduceOp.MIN)[0] > 0.5)
        e2e = {"value": round(nvox / (e2e_ms / 1e3) / 1e9, 3), "unit": UNIT, "steps": e2e_steps,
               "h2d_bytes_per_step": h2d_total, "d2h_bytes_per_step": d2h_total,
               "ms_per_step": round(e2e_ms, 3), "matches_device_result": e2e_ok,
               "path": "apply_filter_host / vkt_apply_filter_host: pinned host slab(+halo) -> "
                       "z-chunks H2D | ApplyFilter | D2H overlapped -> pinned host"}
        del pin_in, pin_out, host_in, host_out, core_in, core_out

    # ---- roofline of the dominant kernel (whole slab at N=1, interior at N>1) ----
    hbm_gbs, sm_max, peak_src = load_peaks()
    props = torch.cuda.get_device_properties(dev)
    local_planes = src.local.dims.z - (2 * kernel.radius.z if world > 1 else 0)
    kvox = nx * ny * local_planes
    kpath = vk.filter_path(dst.local, src.local, kernel, mode)
    roof = roofline_obj(kvox, kern_ms, fmt.bytes_per_cell, algorithmic_fma(kernel, kpath), hbm_gbs, sm_max,
                        props.multi_processor_count)
    roof["traffic"] = None
    roof["peak_source"] = (f"fp32: {props.multi_processor_count} SMs x 128 FMA/clk x {sm_max:.0f} MHz "
                           f"(sm_max_mhz, {peak_src}); hbm: {hbm_gbs} GB/s {peak_src}")
    roof["kernel_ms"] = round(kern_ms, 4)
    roof["kernel_path"] = kpath
    roof["algorithmic_per_voxel"] = {"bytes": 2 * fmt.bytes_per_cell, "fma": algorithmic_fma(kernel, kpath)}
    if kpath == "separable":
        roof["algorithm"] = ("rank-1 weights as three fused 1-D passes (csrc/filter_sep.cuh): "
                             f"{algorithmic_fma(kernel, kpath)} FMAs per voxel instead of {kernel.tap_count}")
        # the dense correlation's own bound (every tap at FP32 peak, or HBM)
        # over this kernel's time: > 1 means faster than any dense kernel can be
        dense_ideal = roofline_obj(kvox, 1.0, fmt.bytes_per_cell, kernel.tap_count, hbm_gbs, sm_max,
                                   props.multi_processor_count)["frac"]  # = ideal ms at 1 ms
        roof["vs_dense_roofline"] = round(dense_ideal / kern_ms, 3)
    tf = ROOT / "profiles" / "ncu_traffic.json"
    ncu_ns = None
    if tf.exists():
        table = json.loads(tf.read_text())
        ent = table.get(f"{args.config} 1 GPU")
        ent = table.get(f"{args.config} 1 GPU {kpath}", ent if kpath == "tma" else None)
        if ent and world == 1:
            roof["traffic"] = ent["total_bytes"]
            roof["traffic_note"] = (f"dram read+write per launch from {ent['capture']} "
                                    f"(algorithmic {ent['algorithmic_bytes']} B)")
        # ncu-measured achieved DRAM GB/s (3^3) and FMA-pipe utilisation (7^3)
        # of the north-star kernels, from the committed captures (a number
        # taken under ncu is never a bench value; these explain the rates)
        ncu_ns = table.get("north_star_ncu")
        if ncu_ns:
            ncu_ns = dict(ncu_ns, peaks={"hbm_gbs": hbm_gbs, "fma_pipe_pct": 100.0})

    # The same workload on the dense tiled kernel (FilterPath.DENSE, every
    # tap evaluated, bit-identical to the direct kernel): the FP32 FMA-pipe
    # utilisation the north star quotes for 7^3.
    dense = None
    if world == 1 and not args.no_extra and kpath == "separable":
        dms, dv, dpath = kernel_rate(kernel, (nx, ny, nz), reps=5, fmt=fmt, path="dense", mode=mode)
        dense = {"path": dpath, "ms": round(dms, 4), "gvox_s": round(dv / dms / 1e6, 2),
                 "roofline": roofline_obj(dv, dms, fmt.bytes_per_cell, kernel.tap_count, hbm_gbs, sm_max,
                                          props.multi_processor_count)}

    extra = None
    if world == 1 and not args.no_extra:
        extra = []
        for name, k in (("gauss3", vk.gaussian_kernel(1.0, 3)), ("box5", vk.box_kernel(5)),
                        ("gauss7", vk.gaussian_kernel(1.5))):
            for path in ("auto", "dense") if k.dims[0] > 3 else ("auto",):
                kms, kv, kp = kernel_rate(k, path=path)
                r = roofline_obj(kv, kms, 4, algorithmic_fma(k, kp), hbm_gbs, sm_max, props.multi_processor_count)
                extra.append({"kernel": name, "dims": [1024, 1024, 1024], "format": "f32",
                              "ms": round(kms, 4), "gvox_s": round(kv / kms / 1e6, 2),
                              "path": kp, "roofline": r})

    # At N > 1, rank 0 also times the unsharded launch over the whole volume
    # (it fits one B200: 2 x 2.1 GB for cfg3, 2 x 34 GB for cfg4) so the line
    # carries the parallel efficiency T1 / (N * T_N) next to the per-rank
    # phases.  (The driver computes its own from the N = 1 run.)
    t1 = None
    if world > 1 and rank == 0 and not args.test_single_gpu and not args.no_t1:
        whole = vk.synthetic_device((nx, ny, nz), fmt, seed=7, device=dev)
        out1 = vk.StructuredVolume(whole.dims, fmt, data=vk.DeviceBuffer(whole.nbytes, device=dev, zero=False))
        for _ in range(2):
            vk.ApplyFilter(out1, whole, kernel, mode)
        ts = []
        for _ in range(3):
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record(stream)
            vk.ApplyFilter(out1, whole, kernel, mode)
            b.record(stream)
            b.synchronize()
            ts.append(a.elapsed_time(b))
        t1 = min(ts)
        del whole, out1
        torch.cuda.empty_cache()

    cpu = None
    if world == 1 and rank == 0 and not args.no_cpu:
        cv, info = cpu_reference(args.config, args.cpu_budget, 1, 0)
        cpu = {"value": round(cv, 6), "unit": UNIT, "cores": info["cores"], "kind": info["kind"],
               "sample": info["sample"]}

    if rank == 0:
        line = {
            "metric": METRIC, "value": round(value, 3), "unit": UNIT, "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": round(ms_step, 4),
            "higher_is_better": True, "scaling": "strong", "vs_baseline": None,
            "dtype": "f32",
            "data": "synthetic (counter-hash, the reference generator's distribution, identical at any N)",
            "config": config_dict(args.config, world),
            "l2": "inputs larger than L2 (no flush between steps)",
            "e2e": e2e,
            "gpu_launches": int(launches),
            "roofline": roof,
            "dense_kernel": dense,
            "clocks": clk.summary(),
            "cpu_baseline": cpu,
            "north_star_f32_1024": extra,
            "ncu": ncu_ns,
        }
        if world > 1:
            line["per_rank_ms"] = [
                {"rank": r, "step": round(v[0], 4), "interior_kernel": round(v[1], 4),
                 "halo_exchange": round(v[2], 4), "boundary_kernels": round(v[3], 4)}
                for r, v in enumerate(per_rank)]
            if t1 is not None:
                line["t1_ms"] = round(t1, 4)
                line["efficiency_vs_1gpu"] = round(t1 / (world * ms_step), 4)
            line["overlap_note"] = ("halo exchange and boundary launches run on a comm stream "
                                    "beside the interior launch; step ~ max(interior, exchange + boundary)")
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.barrier()
        dist.destroy_process_group()


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=30)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", choices=["ours", "reference"], default="ours")
    ap.add_argument("--config", choices=sorted(CONFIGS), default="cfg3")
    ap.add_argument("--e2e-steps", type=int, default=5)
    ap.add_argument("--cpu-budget", type=float, default=20.0)
    ap.add_argument("--no-extra", action="store_true")
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-t1", action="store_true", help="N > 1: skip the unsharded 1-GPU reference launch")
    ap.add_argument("--test-single-gpu", action="store_true",
                    help="testing only: all ranks on cuda:0 over gloo (numbers are not a benchmark)")
    args = ap.parse_args()
    if args.gpus > 1 and "WORLD_SIZE" not in os.environ:
        sys.exit(spawn_ranks(args.gpus))
    if args.warmup < 3 and args.impl == "ours":
        print("warning: warm-up < 3 steps", file=sys.stderr)
    if args.impl == "reference":
        run_reference(args)
    else:
        run_ours(args)


if __name__ == "__main__":
    main()
