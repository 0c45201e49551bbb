"""Time every BASELINE.json config on one B200 (device-resident, CUDA events).

cfg1 256^3 u8  Gaussian 3^3 Clamp
cfg2 512^3 f32 box 5^3 Mirror
cfg3 1024^3 u16 Gaussian 7^3 Clamp        (the bench workload)
cfg4 2048^3 f32 Laplacian 3^3 Wrap        (single-GPU leg of the 8-GPU config)
cfg5 512^3 u8 teaser: Fill(0.5) -> FillRange([128,384)^3, 1.0) -> Gaussian 5^3, all 4 modes

Prints one JSON line per config with ms, GVox/s and the roofline fraction.
"""

import json
import statistics
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))

import torch

import paper_2203_10213_b200 as vk

HBM = json.loads((Path(__file__).resolve().parent.parent / "MEASURED_PEAKS.json").read_text()).get("hbm_gbs", 6545.3) \
    if (Path(__file__).resolve().parent.parent / "MEASURED_PEAKS.json").exists() else 6545.3
FMA = 148 * 128 * 1965e6


def timeit(fn, reps=20, warm=3):
    s = torch.cuda.current_stream()
    for _ in range(warm):
        fn()
    ts = []
    for _ in range(reps):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(s)
        fn()
        b.record(s)
        b.synchronize()
        ts.append(a.elapsed_time(b))
    return min(ts), statistics.median(ts)


def roof(nvox, bpc, taps, ms):
    t_h = nvox * 2 * bpc / (HBM * 1e9)
    t_f = nvox * taps / FMA
    t = max(t_h, t_f)
    return {"bound": "hbm" if t_h >= t_f else "fp32", "frac": round(t / (ms / 1e3), 4)}


def fmas(kernel, path):
    """FMAs per voxel of the algorithm the path runs (separable: 3 1-D sums)."""
    kx, ky, kz = kernel.dims
    return kx + ky + kz if path == "separable" else kx * ky * kz


def filt(name, n, fmt, kernel, mode, reps=20):
    src = vk.synthetic_device((n, n, n), fmt, seed=7)
    dst = vk.StructuredVolume(src.dims, fmt, data=vk.DeviceBuffer(src.nbytes, zero=False))
    best, med = timeit(lambda: vk.ApplyFilter(dst, src, kernel, mode), reps)
    nvox = n ** 3
    path = vk.filter_path(dst, src, kernel, mode)
    taps = fmas(kernel, path)
    out = {"config": name, "n": n, "format": fmt.short_name, "k": list(kernel.dims), "mode": mode,
           "path": path, "ms_best": round(best, 4),
           "ms_median": round(med, 4), "gvox_s": round(nvox / best / 1e6, 2),
           "roofline": roof(nvox, fmt.bytes_per_cell, taps, best)}
    if n <= 512:
        # small volumes: also the launch replayed from a CUDA graph (device time
        # without the ~15 us of per-call host work)
        st = torch.cuda.current_stream()
        side = torch.cuda.Stream()
        side.wait_stream(st)
        with torch.cuda.stream(side):
            vk.ApplyFilter(dst, src, kernel, mode)
            g = torch.cuda.CUDAGraph()
            with torch.cuda.graph(g, stream=side):
                for _ in range(10):
                    vk.ApplyFilter(dst, src, kernel, mode)
        st.wait_stream(side)
        gb, _ = timeit(g.replay, reps)
        out["graph_ms_per_call"] = round(gb / 10, 4)
        out["graph_roofline"] = roof(nvox, fmt.bytes_per_cell, taps, gb / 10)
    del src, dst
    torch.cuda.empty_cache()
    return out


def teaser(n=512):
    v = vk.create_structured_volume((n, n, n), vk.DataFormat.UINT8)
    dst = vk.StructuredVolume(v.dims, v.format, data=vk.DeviceBuffer(v.nbytes, zero=False))
    k = vk.gaussian_kernel(1.0)
    res = {"config": "cfg5 teaser", "n": n, "format": "u8", "k": [5, 5, 5]}
    res["fill_ms"] = round(timeit(lambda: vk.fill(v, 0.5))[0], 4)
    res["fill_gbs"] = round(n ** 3 / (res["fill_ms"] / 1e3) / 1e9, 1)
    res["fill_range_ms"] = round(timeit(lambda: vk.fill_range(v, ((128,) * 3, (384,) * 3), 1.0))[0], 4)
    for mode in ("wrap", "mirror", "clamp", "border"):
        best, _ = timeit(lambda: vk.ApplyFilter(dst, v, k, mode))
        res[f"{mode}_ms"] = round(best, 4)
    total = res["fill_ms"] + res["fill_range_ms"] + res["clamp_ms"]
    res["pipeline_clamp_ms"] = round(total, 4)
    # the same three calls replayed from a CUDA graph: device time without the
    # per-call host overhead
    st = torch.cuda.current_stream()
    side = torch.cuda.Stream()
    side.wait_stream(st)

    def pipeline():
        vk.fill(v, 0.5)
        vk.fill_range(v, ((128,) * 3, (384,) * 3), 1.0)
        vk.ApplyFilter(dst, v, k, "clamp")

    with torch.cuda.stream(side):
        pipeline()
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g, stream=side):
            pipeline()
    st.wait_stream(side)
    res["pipeline_clamp_graph_ms"] = round(timeit(g.replay)[0], 4)
    res["path"] = vk.filter_path(dst, v, k, "clamp")
    res["filter_roofline_clamp"] = roof(n ** 3, 1, fmas(k, res["path"]), res["clamp_ms"])
    return res


def main():
    U8, U16, F32 = vk.DataFormat.UINT8, vk.DataFormat.UINT16, vk.DataFormat.FLOAT32
    which = sys.argv[1:] or ["1", "2", "3", "4", "5"]
    if "1" in which:
        print(json.dumps(filt("cfg1", 256, U8, vk.gaussian_kernel(1.0, 3), "clamp", reps=50)), flush=True)
    if "2" in which:
        print(json.dumps(filt("cfg2", 512, F32, vk.box_kernel(5), "mirror")), flush=True)
    if "3" in which:
        print(json.dumps(filt("cfg3", 1024, U16, vk.gaussian_kernel(1.5), "clamp", reps=10)), flush=True)
    if "4" in which:
        print(json.dumps(filt("cfg4 (1 GPU)", 2048, F32, vk.laplacian_kernel(), "wrap", reps=5)), flush=True)
    if "5" in which:
        print(json.dumps(teaser()), flush=True)


if __name__ == "__main__":
    main()
