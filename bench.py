#!/usr/bin/env python
"""ApplyFilter benchmark (BASELINE.json metric) — one JSON line on rank 0.

Workload (BASELINE.json configs[2]): 7x7x7 Gaussian (gaussian_kernel(1.5),
SURVEY §8(d)) on a 1024^3 uint16 volume, Clamp (the reference's only mode),
z-slab sharded with NCCL halo exchange at N = 1/2/4/8 GPUs (strong scaling:
the volume is fixed).  A "step" is one ApplyFilter pass over the whole volume.

  python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]

Run multi-GPU as
  python -m torch.distributed.run --nnodes=1 --nproc-per-node N \
      --master-addr 127.0.0.1 --master-port P bench.py --gpus N ...

Timing: W untimed warm-up steps; K timed steps bracketed by a barrier and
cuda synchronize; CUDA events on the launching stream; max over ranks.  The
1024^3 u16 input (2.1 GB; 268 MB per rank at N=8) is larger than the 126 MB
L2, so no flush is needed between steps.  --impl reference times the CPU
oracle port of the reference's apply_filter (oracle/vkt_oracle.py, numpy,
all host threads) on a bounded z-slab sample of the same workload.
"""

from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import time
from pathlib import Path

ROOT = Path(__file__).resolve().parent
sys.path.insert(0, str(ROOT))

METRIC = "ApplyFilter GVoxels/s at 1/2/4/8 B200; % of HBM/FP32 roofline"
UNIT = "GVox/s"
WORKLOAD = dict(workload="cfg3: ApplyFilter 7x7x7 Gaussian(sigma=1.5) on 1024^3 uint16, Clamp, "
                         "z-slab sharded with NCCL halo exchange",
                dims=[1024, 1024, 1024], format="u16", kernel="gaussian_kernel(1.5) 7x7x7",
                address_mode="clamp")


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
        if test_single_gpu:
            dist.init_process_group("gloo")
        else:
            dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    return rank, world, local


def cpu_reference(steps: int, warmup: int, budget_s: float):
    """Oracle port of the reference apply_filter on a bounded z-slab sample."""
    import numpy as np

    from oracle import vkt_oracle as O

    nx = ny = 1024
    w = O.gaussian_weights(1.5)
    rz = w.shape[0] // 2
    cores = len(os.sched_getaffinity(0))
    rng = np.random.default_rng(7)

    def sample(planes):
        # the reference generator's distribution (bench.py:38-48): uniform u16
        vol = rng.integers(0, 65536, size=(planes + 2 * rz, ny, nx), dtype=np.uint16)
        t0 = time.perf_counter()
        O.apply_filter(vol, 2, w, "clamp", z_range=(rz, rz + planes), workers=cores)
        return time.perf_counter() - t0

    t_plane = sample(1)  # calibration (untimed)
    planes = max(1, int(budget_s / max(t_plane, 1e-3)))
    times = []
    for i in range(warmup + steps):
        dt = sample(planes)
        if i >= warmup:
            times.append(dt)
    total = sum(times)
    vox = planes * nx * ny * len(times)
    return vox / total / 1e9, dict(cores=cores, planes=planes, seconds=total,
                                    sample=f"{planes} output planes of 1024x1024 (+{2 * rz} halo) "
                                           f"u16 per step, gaussian 7^3 clamp, {len(times)} steps")


def run_reference(args):
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    steps, warmup = args.steps, args.warmup
    budget = max(0.5, min(20.0, 150.0 / max(1, steps + warmup)))
    value, info = cpu_reference(steps, warmup, budget)
    ms = info["seconds"] / max(1, steps) * 1e3
    line = {
        "metric": METRIC, "value": round(value, 6), "unit": UNIT, "impl": "reference",
        "n_gpus": args.gpus, "steps": steps, "warmup": warmup, "ms_per_step": round(ms, 3),
        "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "f64",
        "data": "synthetic (numpy default_rng(7), uniform u16)",
        "config": dict(WORKLOAD, parallelism="host threads (oracle port of filters.py:69-95)"),
        "cpu_baseline": {"value": round(value, 6), "unit": UNIT, "cores": info["cores"],
                         "kind": "port", "sample": info["sample"]},
        "e2e": {"value": round(value, 6), "unit": UNIT, "h2d_bytes_per_step": 0,
                "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


def kernel_rate_f32(k_name, weights_kernel, dims=(1024, 1024, 1024), reps=10):
    """North-star extra: 1024^3 f32 ApplyFilter kernel time (events, best of reps)."""
    import torch

    import paper_2203_10213_b200 as vk

    src = vk.synthetic_device(dims, vk.DataFormat.FLOAT32, seed=11)
    dst = vk.StructuredVolume(src.dims, src.format, data=vk.DeviceBuffer(src.nbytes, zero=False))
    s = torch.cuda.current_stream()
    for _ in range(2):
        vk.ApplyFilter(dst, src, weights_kernel)
    times = []
    for _ in range(reps):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(s)
        vk.ApplyFilter(dst, src, weights_kernel)
        e1.record(s)
        e1.synchronize()
        times.append(e0.elapsed_time(e1))
    ms = statistics.median(times)
    nvox = dims[0] * dims[1] * dims[2]
    path = vk.filter_path(dst, src, weights_kernel)
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
    import torch
    import torch.distributed as dist

    import paper_2203_10213_b200 as vk
    from paper_2203_10213_b200 import _capi
    from paper_2203_10213_b200.shard import ShardedVolume, apply_filter_sharded

    rank, world, local = dist_setup(args.gpus, args.test_single_gpu)
    dev = torch.device("cuda", local)
    nx, ny, nz = WORKLOAD["dims"]
    fmt = vk.DataFormat.UINT16
    kernel = vk.gaussian_kernel(1.5)
    mode = vk.AddressMode.CLAMP
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

    def barrier():
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize(dev)

    for _ in range(args.warmup):
        apply_filter_sharded(dst, src, kernel, mode, group=group, exchange=exchange)
    barrier()

    launches0 = _capi.launch_count()
    kev = []
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with ClockSampler(local) as clk:
        barrier()
        e0.record(stream)
        for _ in range(args.steps):
            apply_filter_sharded(dst, src, kernel, mode, group=group, exchange=exchange,
                                 kernel_events=kev)
        e1.record(stream)
        barrier()
    launches = _capi.launch_count() - launches0
    ms_total = e0.elapsed_time(e1)
    kern_ms = statistics.mean(a.elapsed_time(b) for a, b in kev)
    ms_total, kern_ms = allreduce([ms_total, kern_ms], dist.ReduceOp.MAX)
    ms_step = ms_total / args.steps
    nvox = nx * ny * nz
    value = nvox / (ms_step / 1e3) / 1e9

    # ---- e2e through the public API with host buffers (pinned) ----
    # vkt_apply_filter_host (paper_2203_10213_b200.apply_filter_host): each
    # rank passes its halo-extended z-slab of the host volume (what range I/O
    # would read); the library streams z-chunks H2D -> filter -> D2H with the
    # three phases overlapped.  Every step moves the slab + halos in and the
    # slab out.
    import numpy as np

    e2e_steps = max(1, min(args.steps, args.e2e_steps))
    rz = kernel.radius.z
    lo, hi = max(0, src.z0 - rz), min(nz, src.z1 + rz)
    plane_b = nx * ny * fmt.bytes_per_cell
    pin_in = torch.empty((hi - lo) * plane_b, dtype=torch.uint8, pin_memory=True)
    pin_out = torch.empty((hi - lo) * plane_b, dtype=torch.uint8, pin_memory=True)
    pin_in[(src.z0 - lo) * plane_b:(src.z1 - lo) * plane_b].copy_(src.local.data.array)
    if src.z0 > lo or hi > src.z1:  # halo planes of the host copy: regenerate on device
        for (g0, g1) in ((lo, src.z0), (src.z1, hi)):
            if g1 > g0:
                h = vk.synthetic_device((nx, ny, nz), fmt, seed=7, z_offset=g0, local_nz=g1 - g0, device=dev)
                pin_in[(g0 - lo) * plane_b:(g1 - lo) * plane_b].copy_(h.data.array)
    host_in = pin_in.numpy().view(fmt.dtype).reshape(hi - lo, ny, nx)
    host_out = pin_out.numpy().view(fmt.dtype).reshape(hi - lo, ny, nx)
    # untimed warm-up: the first call grows the library's device pool (the
    # resident padded input, > 2 GB at cfg3) — a one-time cost, not a step
    for _ in range(min(args.warmup, 2)):
        vk.apply_filter_host(host_in, kernel, mode, out=host_out, z_offset=lo, global_nz=nz,
                             z_range=(src.z0 - lo, src.z1 - lo))
    torch.cuda.synchronize()
    barrier()
    f0, f1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    f0.record(stream)
    for _ in range(e2e_steps):
        vk.apply_filter_host(host_in, kernel, mode, out=host_out, z_offset=lo, global_nz=nz,
                             z_range=(src.z0 - lo, src.z1 - lo))
    f1.record(stream)
    barrier()
    e2e_ms = allreduce([f0.elapsed_time(f1)], dist.ReduceOp.MAX)[0] / e2e_steps
    e2e_value = nvox / (e2e_ms / 1e3) / 1e9
    # host result must equal the device-resident result
    e2e_ok = bool(torch.equal(pin_out[(src.z0 - lo) * plane_b:(src.z1 - lo) * plane_b],
                              dst.local.data.array.cpu()))
    h2d_bytes = (hi - lo) * plane_b
    d2h_bytes = (src.z1 - src.z0) * plane_b
    h2d_total, d2h_total = (int(v) for v in allreduce([h2d_bytes, d2h_bytes], dist.ReduceOp.SUM))
    e2e_ok = bool(allreduce([1.0 if e2e_ok else 0.0], dist.ReduceOp.MIN)[0] > 0.5)
    del np

    # ---- roofline of the dominant kernel (interior launch on each rank) ----
    hbm_gbs, sm_max, peak_src = load_peaks()
    props = torch.cuda.get_device_properties(dev)
    local_planes = src.local.dims.z - (2 * kernel.radius.z if world > 1 else 0)
    kvox = nx * ny * local_planes
    roof = roofline_obj(kvox, kern_ms, fmt.bytes_per_cell, kernel.tap_count, hbm_gbs, sm_max,
                        props.multi_processor_count)
    roof["traffic"] = None
    roof["peak_source"] = (f"fp32: {props.multi_processor_count} SMs x 128 FMA/clk x {sm_max:.0f} MHz "
                           f"(sm_max_mhz, {peak_src}); hbm: {hbm_gbs} GB/s {peak_src}")
    roof["kernel_ms"] = round(kern_ms, 4)
    roof["kernel_path"] = vk.filter_path(dst.local, src.local, kernel)
    tf = ROOT / "profiles" / "ncu_traffic.json"
    if tf.exists() and world == 1 and roof["kernel_path"] == "tma":
        ent = json.loads(tf.read_text()).get("filter_tma_kernel<u16,7,clamp> 1024^3")
        if ent:
            roof["traffic"] = ent["total_bytes"]
            roof["traffic_note"] = (f"dram read+write per launch from {ent['capture']} "
                                    f"(algorithmic {ent['algorithmic_bytes']} B)")
    # ncu-measured achieved DRAM GB/s (3^3) and FMA-pipe utilisation (7^3) of
    # the north-star kernels, from the committed captures (a number taken
    # under ncu is never a bench value; these explain the CUDA-event rates)
    ncu_ns = None
    if tf.exists():
        ncu_ns = json.loads(tf.read_text()).get("north_star_ncu")
        if ncu_ns:
            ncu_ns = dict(ncu_ns, peaks={"hbm_gbs": hbm_gbs, "fma_pipe_pct": 100.0})

    extra = None
    if world == 1 and not args.no_extra:
        extra = []
        for name, k in (("gauss3", vk.gaussian_kernel(1.0, 3)), ("box5", vk.box_kernel(5)),
                        ("gauss7", vk.gaussian_kernel(1.5))):
            kms, kv, kpath = kernel_rate_f32(name, k)
            r = roofline_obj(kv, kms, 4, k.tap_count, hbm_gbs, sm_max, props.multi_processor_count)
            extra.append({"kernel": name, "dims": [1024, 1024, 1024], "format": "f32",
                          "ms": round(kms, 4), "gvox_s": round(kv / kms / 1e6, 2),
                          "path": kpath, "roofline": r})

    cpu = None
    if world == 1 and rank == 0 and not args.no_cpu:
        cv, info = cpu_reference(1, 0, args.cpu_budget)
        cpu = {"value": round(cv, 6), "unit": UNIT, "cores": info["cores"], "kind": "port",
               "sample": info["sample"]}

    if rank == 0:
        line = {
            "metric": METRIC, "value": round(value, 3), "unit": UNIT, "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": round(ms_step, 4),
            "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "f32",
            "data": "synthetic (counter-hash, uniform u16 over [0, 65535], identical at any N)",
            "config": dict(WORKLOAD, parallelism=f"z-slab x{world}",
                           l2="inputs larger than L2 (2.1 GB total, >= 268 MB per rank); no flush"),
            "e2e": {"value": round(e2e_value, 3), "unit": UNIT, "steps": e2e_steps,
                    "h2d_bytes_per_step": h2d_total, "d2h_bytes_per_step": d2h_total,
                    "ms_per_step": round(e2e_ms, 3), "matches_device_result": e2e_ok,
                    "path": "apply_filter_host / vkt_apply_filter_host: pinned host slab(+halo) -> "
                            "z-chunks H2D | ApplyFilter | D2H overlapped -> pinned host"},
            "gpu_launches": int(launches),
            "roofline": roof,
            "clocks": clk.summary(),
            "cpu_baseline": cpu,
            "north_star_f32_1024": extra,
            "ncu": ncu_ns,
        }
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
    ap.add_argument("--e2e-steps", type=int, default=5)
    ap.add_argument("--cpu-budget", type=float, default=15.0)
    ap.add_argument("--no-extra", action="store_true")
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--test-single-gpu", action="store_true",
                    help="testing only: all ranks on cuda:0 over gloo (numbers are not a benchmark)")
    args = ap.parse_args()
    if args.warmup < 3 and args.impl == "ours":
        print("warning: warm-up < 3 steps", file=sys.stderr)
    if args.impl == "reference":
        run_reference(args)
    else:
        run_ours(args)


if __name__ == "__main__":
    main()
