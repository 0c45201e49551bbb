"""Rates of the SURVEY §8(f) rows on the B200 beside the reference's CPU path.

Device side: CUDA events around each call on a device-resident volume (best
of N), throughput in GVox/s and the HBM fraction of its algorithmic bytes
(bytes read + written once).  Reference side: the unmodified reference
(baseline/_ref, the same functions through its public API) on a smaller
sample, all host threads, best of 2 — context only.  I/O: VKTVOL01 read /
write through the page cache (/tmp), and filter_file end to end.

  python tools/next_rows_rates.py > profiles/r02_next_rows_rates.jsonl
"""

import json
import os
import sys
import tempfile
import time
from pathlib import Path

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))

HBM = json.loads((ROOT / "MEASURED_PEAKS.json").read_text()).get("hbm_gbs", 6541.5) \
    if (ROOT / "MEASURED_PEAKS.json").exists() else 6541.5


def dev_time(fn, reps=10, warm=2):
    import torch

    s = torch.cuda.current_stream()
    for _ in range(warm):
        fn()
    best = 1e9
    for _ in range(reps):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(s)
        fn()
        b.record(s)
        b.synchronize()
        best = min(best, a.elapsed_time(b))
    return best


def ref_time(fn, reps=2):
    best = 1e9
    for _ in range(reps):
        t = time.perf_counter()
        fn()
        best = min(best, time.perf_counter() - t)
    return best * 1e3


def _reference():
    ref = ROOT / "baseline" / "_ref"
    if not (ref / "vkt").exists():
        return None
    sys.path.insert(0, str(ref))
    import vkt  # noqa: E402

    return vkt


def line(**kw):
    print(json.dumps(kw), flush=True)


def main():
    import numpy as np
    import torch

    import paper_2203_10213_b200 as vk

    rv = _reference()
    U8 = vk.DataFormat.UINT8
    n = 512
    nvox = n ** 3

    # Flip (geometric.py:34-40): read + write every cell once
    v = vk.synthetic_device((n, n, n), U8, seed=7)
    ms = dev_time(lambda: vk.flip(v, 0))
    row = dict(op="flip axis 0", dims=[n] * 3, format="u8", ms=round(ms, 4), gvox_s=round(nvox / ms / 1e6, 1),
               hbm_frac=round(2 * nvox / (ms / 1e3) / 1e9 / HBM, 3))
    if rv:
        m = 256
        rvol = rv.synthetic_structured(m, rv.DataFormat.UINT8)
        rms = ref_time(lambda: rv.flip(rvol, 0))
        row["reference_cpu"] = {"dims": [m] * 3, "ms": round(rms, 2), "gvox_s": round(m ** 3 / rms / 1e6, 4)}
    line(**row)

    # Resample down by 2 (core.py:202-262): read src once, write dst
    ms = dev_time(lambda: vk.resample(v, (n // 2,) * 3), reps=10)
    out_vox = (n // 2) ** 3
    row = dict(op="resample to half", dims=[n] * 3, format="u8", ms=round(ms, 4),
               gvox_s_out=round(out_vox / ms / 1e6, 1),
               hbm_frac=round((nvox + out_vox) / (ms / 1e3) / 1e9 / HBM, 3))
    if rv:
        m = 128
        rvol = rv.synthetic_structured(m, rv.DataFormat.UINT8)
        rms = ref_time(lambda: rv.resample(rvol, (m // 2,) * 3))
        row["reference_cpu"] = {"dims": [m] * 3, "ms": round(rms, 2), "gvox_s_out": round((m // 2) ** 3 / rms / 1e6, 4)}
    line(**row)

    # FillRange (core.py:39-55): write the box once
    lo, hi = (n // 4,) * 3, (3 * n // 4,) * 3
    box = (n // 2) ** 3
    ms = dev_time(lambda: vk.fill_range(v, (lo, hi), 0.5))
    row = dict(op="fill_range half box", dims=[n] * 3, format="u8", ms=round(ms, 4),
               gvox_s=round(box / ms / 1e6, 1), hbm_frac=round(box / (ms / 1e3) / 1e9 / HBM, 3))
    if rv:
        m = 256
        rvol = rv.synthetic_structured(m, rv.DataFormat.UINT8)
        rms = ref_time(lambda: rv.fill_range(rvol, rv.box3i((m // 4,) * 3, (3 * m // 4,) * 3), 0.5))
        row["reference_cpu"] = {"dims": [m] * 3, "ms": round(rms, 2), "gvox_s": round((m // 2) ** 3 / rms / 1e6, 4)}
    line(**row)

    # CLAHE-3D (filters.py:101-190): histogram pass reads every cell, blend
    # pass reads + writes every cell
    m = 256
    cv = vk.synthetic_device((m, m, m), U8, seed=7)
    params = vk.ClaheParams((4, 4, 4), 256, 3.0)
    ms = dev_time(lambda: vk.clahe_equalize(cv, params), reps=5)
    row = dict(op="clahe_equalize bricks 4^3, 256 bins, clip 3", dims=[m] * 3, format="u8", ms=round(ms, 4),
               gvox_s=round(m ** 3 / ms / 1e6, 2), hbm_frac=round(3 * m ** 3 / (ms / 1e3) / 1e9 / HBM, 3))
    if rv:
        mm = 128
        rvol = rv.synthetic_structured(mm, rv.DataFormat.UINT8)
        rms = ref_time(lambda: rv.clahe_equalize(rvol, rv.ClaheParams((4, 4, 4), 256, 3.0)))
        row["reference_cpu"] = {"dims": [mm] * 3, "ms": round(rms, 2), "gvox_s": round(mm ** 3 / rms / 1e6, 4)}
    line(**row)
    del cv

    # VKTVOL01 I/O through the page cache, and filter_file end to end
    tmp = Path(tempfile.mkdtemp())
    f_in, f_out = tmp / "in.vkt", tmp / "out.vkt"
    n2 = 512
    big = vk.synthetic_device((n2, n2, n2), vk.DataFormat.UINT16, seed=7)
    vk.write_volume(f_in, big)
    nbytes = n2 ** 3 * 2
    t = time.perf_counter()
    vk.write_volume(f_in, big)
    torch.cuda.synchronize()
    w_s = time.perf_counter() - t
    t = time.perf_counter()
    r = vk.read_volume(f_in)
    torch.cuda.synchronize()
    r_s = time.perf_counter() - t
    line(op="write_volume / read_volume (VKTVOL01, page cache)", dims=[n2] * 3, format="u16",
         write_gbs=round(nbytes / w_s / 1e9, 2), read_gbs=round(nbytes / r_s / 1e9, 2))
    del r
    k = vk.gaussian_kernel(1.5)
    vk.filter_file(f_in, f_out, k, "clamp")
    t = time.perf_counter()
    vk.filter_file(f_in, f_out, k, "clamp")
    ff_s = time.perf_counter() - t
    line(op="filter_file Gaussian 7^3 Clamp (file -> B200 -> file, out of core)", dims=[n2] * 3, format="u16",
         s=round(ff_s, 3), gvox_s=round(n2 ** 3 / ff_s / 1e9, 3))
    for f in (f_in, f_out):
        os.unlink(f)
    os.rmdir(tmp)


if __name__ == "__main__":
    main()
