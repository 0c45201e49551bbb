"""TEST INFRASTRUCTURE ONLY — generate tests/golden/*.npz from the REAL reference.

Run in the build container (where /root/reference exists):

    PYTHONPATH=/root/reference/pkg/src python oracle/make_golden.py

It imports the reference package ``vkt`` read-only and records, for a matrix
of small seeded volumes, the reference's own outputs:
  * clamp cases: ``vkt.apply_filter`` verbatim (filters.py:69-95);
  * wrap / mirror / border cases: the reference-anchored construction of
    SURVEY.md §8(c) — pad the stored cells with np.pad(mode), run the
    reference apply_filter on the padded volume, crop the centre;
  * fill cases: ``vkt.fill_range`` (core.py:39-55).
The fixtures are committed; the GPU box never needs /root/reference.
"""

from __future__ import annotations

import sys
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parent.parent
OUT = ROOT / "tests" / "golden"

sys.path.insert(0, "/root/reference/pkg/src")
import vkt  # noqa: E402  (the reference, read-only)
from vkt.ops.filters import box_kernel  # noqa: E402

FMTS = {1: vkt.DataFormat.UINT8, 2: vkt.DataFormat.UINT16, 3: vkt.DataFormat.FLOAT32}
PAD = {"wrap": "wrap", "mirror": "symmetric", "border": "constant"}


def random_stored(rng, dims, fmt):
    nx, ny, nz = dims
    if fmt == 3:
        return rng.random((nz, ny, nx), dtype=np.float32)
    dt = np.uint8 if fmt == 1 else np.uint16
    return rng.integers(0, np.iinfo(dt).max + 1, size=(nz, ny, nx), dtype=dt)


def reference_filter(stored, fmt, mapping, kernel, mode):
    nz, ny, nx = stored.shape
    if mode == "clamp":
        v = vkt.StructuredVolume((nx, ny, nz), FMTS[fmt], (1, 1, 1), mapping)
        v.array()[...] = stored
        vkt.apply_filter(v, kernel)
        return v.array().copy()
    r = kernel.radius
    p = np.pad(stored, ((r.z, r.z), (r.y, r.y), (r.x, r.x)), mode=PAD[mode])
    big = vkt.StructuredVolume(p.shape[::-1], FMTS[fmt], (1, 1, 1), mapping)
    big.array()[...] = p
    vkt.apply_filter(big, kernel)
    return big.array()[r.z:r.z + nz, r.y:r.y + ny, r.x:r.x + nx].copy()


def kernels(rng):
    aniso = rng.normal(size=15)
    yield "gauss3", vkt.gaussian_kernel(1.0, 3)
    yield "gauss5", vkt.gaussian_kernel(1.0)
    yield "gauss7", vkt.gaussian_kernel(1.5)
    yield "box5", box_kernel(5)
    lap = np.zeros((3, 3, 3))
    lap[1, 1, 1] = -6.0
    for z, y, x in ((0, 1, 1), (2, 1, 1), (1, 0, 1), (1, 2, 1), (1, 1, 0), (1, 1, 2)):
        lap[z, y, x] = 1.0
    yield "lap3", vkt.Kernel((3, 3, 3), lap)
    yield "aniso315", vkt.Kernel((3, 1, 5), aniso / np.abs(aniso).sum())
    yield "ident1", vkt.Kernel((1, 1, 1), [1.0])
    yield "rand3", vkt.Kernel((3, 3, 3), rng.normal(size=27) * 0.2)


def main():
    OUT.mkdir(parents=True, exist_ok=True)
    rng = np.random.default_rng(20220321)
    cases = {}
    idx = 0
    shapes = [(13, 11, 9), (6, 5, 7), (2, 3, 4), (1, 1, 5), (17, 4, 3)]
    for kname, kernel in kernels(rng):
        for fmt in (1, 2, 3):
            mappings = [(0.0, 1.0)] if fmt == 3 else [(0.0, 1.0), (-1.0, 3.0)]
            for mapping in mappings:
                for mode in ("clamp", "wrap", "mirror", "border"):
                    dims = shapes[idx % len(shapes)]
                    idx += 1
                    stored = random_stored(rng, dims, fmt)
                    out = reference_filter(stored, fmt, mapping, kernel, mode)
                    key = f"c{idx:04d}"
                    cases[f"{key}/input"] = stored
                    cases[f"{key}/output"] = out
                    cases[f"{key}/weights"] = kernel.weights
                    cases[f"{key}/meta"] = np.array(
                        [fmt, mapping[0], mapping[1], ("wrap", "mirror", "clamp", "border").index(mode)],
                        dtype=np.float64)
                    cases[f"{key}/name"] = np.array(f"{kname}/{FMTS[fmt].short_name}/{mapping}/{mode}")
    np.savez_compressed(OUT / "filter_cases.npz", **cases)

    # bench-shaped fixture: the reference generator at seed 7 (bench.py:38-48)
    # on a 24^3 u8 cube through gaussian_kernel(1.0, 3), the bench's kernel (bench.py:97)
    v = vkt.synthetic_structured(24, vkt.DataFormat.UINT8, 7)
    before = v.array().copy()
    vkt.apply_filter(v, vkt.gaussian_kernel(1.0, 3))
    np.savez_compressed(OUT / "bench_case.npz", input=before, output=v.array().copy())

    # fill cases (core.py:39-55): (dims, fmt, mapping, roi lower, roi upper, value)
    fills = {}
    frng = np.random.default_rng(99)
    specs = [
        ((64, 64, 64), 1, (0.0, 1.0), (1, 1, 1), (63, 63, 63), 1.0),   # Fig. 4 session
        ((8, 8, 8), 1, (0.0, 1.0), (0, 0, 0), (8, 8, 8), 0.5),
        ((6, 6, 6), 1, (0.0, 1.0), (1, 2, 3), (4, 5, 6), 0.25),
        ((4, 4, 4), 1, (0.0, 1.0), (-5, -5, -5), (99, 99, 99), 1.0),
        ((9, 7, 5), 2, (-1.0, 3.0), (2, 0, 1), (9, 7, 4), 0.3337),
        ((9, 7, 5), 3, (0.0, 1.0), (3, 1, 0), (7, 6, 5), -2.5),
        ((33, 5, 4), 1, (0.0, 1.0), (1, 1, 1), (32, 4, 3), 0.7),
        ((33, 5, 4), 2, (0.0, 1.0), (0, 0, 0), (33, 5, 4), 2.0),
        ((4, 4, 4), 2, (0.0, 1.0), (2, 2, 2), (2, 2, 2), 1.0),          # empty roi
        ((31, 3, 2), 3, (0.0, 1.0), (5, 0, 0), (31, 3, 2), 0.1),
    ]
    for i, (dims, fmt, mapping, lower, upper, value) in enumerate(specs):
        stored = random_stored(frng, dims, fmt)
        if i == 0:  # the Fig. 4 session starts from a zero-filled volume
            stored = np.zeros_like(stored)
        v = vkt.StructuredVolume(dims, FMTS[fmt], (1, 1, 1), mapping)
        v.array()[...] = stored
        vkt.fill_range(v, vkt.box3i(lower, upper), value)
        fills[f"f{i:02d}/input"] = stored
        fills[f"f{i:02d}/output"] = v.array().copy()
        fills[f"f{i:02d}/spec"] = np.array([fmt, mapping[0], mapping[1], *lower, *upper, value])
    np.savez_compressed(OUT / "fill_cases.npz", **fills)

    # VKTVOL01 files written by the reference (io.py:164-194) and the output
    # of the reference CLI `vkt filter` on them (cli.py:359-375)
    import subprocess
    vrng = np.random.default_rng(5)
    for fmt, dims, mapping, cell in ((1, (20, 12, 9), (0.0, 1.0), (1.0, 1.0, 1.0)),
                                    (2, (16, 8, 11), (-1.0, 3.0), (0.5, 1.0, 2.0)),
                                    (3, (12, 10, 7), (0.0, 1.0), (1.0, 1.0, 1.0))):
        v = vkt.StructuredVolume(dims, FMTS[fmt], cell, mapping)
        v.array()[...] = random_stored(vrng, dims, fmt)
        name = f"vol_{FMTS[fmt].short_name}.vkt"
        vkt.write_volume(OUT / name, v)
        out = subprocess.run([sys.executable, "-m", "vkt", "filter", "--gaussian", "1.0", "--ksize", "3",
                              "-i", str(OUT / name), "-o", str(OUT / f"filtered_{name}")],
                             env={**__import__("os").environ, "PYTHONPATH": "/root/reference/pkg/src"},
                             capture_output=True)
        assert out.returncode == 0, out.stderr

    # CLAHE-3D (filters.py:98-245): reference outputs and brick mappings
    import math
    crng = np.random.default_rng(2203)
    clahe = {}
    cspecs = [((16, 16, 16), 1, (0.0, 1.0), (2, 2, 2), 64, 3.0),
              ((20, 12, 9), 1, (0.0, 1.0), (1, 1, 1), 256, math.inf),
              ((17, 13, 11), 2, (-1.0, 3.0), (3, 2, 2), 128, 2.5),
              ((12, 10, 7), 3, (0.0, 1.0), (2, 3, 1), 32, math.inf),
              ((32, 32, 32), 1, (-1.0, 2.0), (2, 2, 2), 256, 4.0),
              ((9, 21, 5), 3, (-0.5, 1.5), (2, 4, 3), 50, 1.0),
              ((256, 1, 1), 1, (0.0, 1.0), (1, 1, 1), 256, math.inf)]
    for i, (dims, fmt, mapping, bricks, bins, clip) in enumerate(cspecs):
        stored = random_stored(crng, dims, fmt)
        if i == len(cspecs) - 1:
            stored = np.arange(256, dtype=np.uint8).reshape(1, 1, 256)
        v = vkt.StructuredVolume(dims, FMTS[fmt], (1, 1, 1), mapping)
        v.array()[...] = stored
        params = vkt.ClaheParams(bricks, bins, clip)
        from vkt.ops.filters import brick_mappings
        maps = brick_mappings(v, params)
        vkt.clahe_equalize(v, params)
        clahe[f"h{i:02d}/input"] = stored
        clahe[f"h{i:02d}/output"] = v.array().copy()
        clahe[f"h{i:02d}/maps"] = maps
        clahe[f"h{i:02d}/spec"] = np.array([fmt, mapping[0], mapping[1], *bricks, bins, clip])
    np.savez_compressed(OUT / "clahe_cases.npz", **clahe)

    # Resample / Flip (ops/core.py:202-262, ops/geometric.py:34-40)
    xrng = np.random.default_rng(523)
    xf = {}
    rspecs = [((16, 12, 10), 1, (0.0, 1.0), (8, 6, 5), 1, (0.0, 1.0)),
              ((13, 9, 7), 2, (-1.0, 3.0), (20, 4, 11), 3, (0.0, 1.0)),
              ((10, 10, 10), 3, (0.0, 1.0), (7, 13, 3), 2, (-0.5, 1.5)),
              ((1, 5, 3), 1, (0.0, 1.0), (4, 2, 6), 1, (0.0, 1.0)),
              ((24, 24, 24), 3, (0.0, 1.0), (12, 12, 12), 3, (0.0, 1.0))]
    for i, (dims, fmt, mapping, ddims, dfmt, dmap) in enumerate(rspecs):
        stored = random_stored(xrng, dims, fmt)
        v = vkt.StructuredVolume(dims, FMTS[fmt], (1, 0.5, 2), mapping)
        v.array()[...] = stored
        r = vkt.resample(v, ddims, FMTS[dfmt], dmap)
        xf[f"r{i}/input"] = stored
        xf[f"r{i}/output"] = r.array().copy()
        xf[f"r{i}/spec"] = np.array([fmt, *mapping, *ddims, dfmt, *dmap])
        xf[f"r{i}/cell"] = np.array(tuple(r.cell_size))
        for ax in range(3):
            f = v.copy()
            vkt.flip(f, ax)
            xf[f"r{i}/flip{ax}"] = f.array().copy()
    np.savez_compressed(OUT / "transform_cases.npz", **xf)
    print(f"wrote {idx} filter cases, {len(specs)} fill cases, 3 VKTVOL01 files, {len(cspecs)} CLAHE cases to {OUT}")


if __name__ == "__main__":
    main()
