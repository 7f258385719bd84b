"""Generate golden SF fixtures by running the REAL reference package.

Run in the build container (where /root/reference exists):

    PYTHONDONTWRITEBYTECODE=1 NUMBA_CACHE_DIR=/tmp/numba_cache \
        python tests/golden/make_golden.py

It imports ``ctproj`` from /root/reference/pkg/src (numba, read-only), runs
``sf_forward`` / ``sf_backproject`` (pkg/src/ctproj/sf.py:30-45) on seeded
inputs and writes ``tests/golden/sf_golden.npz``.  Nothing on the GPU box reads
/root/reference; tests only read the committed .npz.

Each case stores the config (reference JSON key format, as parse_config
accepts it, geometry.py:431-512), the f32 inputs and the reference f32
outputs.  ``explicit_*`` cases store the explicit forward matrix A (columns =
unit-volume responses) and the explicit back matrix B (columns = unit-sinogram
responses) for the transpose test of pkg/tests/test_sf.py:89-111.
"""

from __future__ import annotations

import json
import os
import sys

import numpy as np

REF = "/root/reference/pkg/src"
OUT = os.path.join(os.path.dirname(os.path.abspath(__file__)), "sf_golden.npz")


def cases():
    c = {}
    # pkg/tests/conftest.py:71-75 fixtures (parallel_small / cone_small) + curved
    base = dict(numX=12, numY=12, numZ=12, voxelWidth=1.25, voxelHeight=1.25)
    c["parallel_small"] = dict(base, geometry="parallel", numRows=16, numCols=16,
                               pixelHeight=1.25, pixelWidth=1.25,
                               angles=[180.0 * i / 8 for i in range(8)])
    c["cone_small"] = dict(base, geometry="cone", numRows=16, numCols=16,
                           pixelHeight=2.0, pixelWidth=2.0, sod=40.0, sdd=80.0,
                           angles=[360.0 * i / 8 for i in range(8)])
    c["curved_small"] = dict(c["cone_small"], geometry="cone-curved")
    # offsets, shifted detector centre, anisotropic pixels, non-cubic grid,
    # irregular angle list
    c["offset_cone"] = dict(geometry="cone", numX=10, numY=14, numZ=6,
                            voxelWidth=1.0, voxelHeight=1.3,
                            offsetX=0.8, offsetY=-0.4, offsetZ=0.2,
                            numRows=12, numCols=20, pixelHeight=1.1, pixelWidth=0.9,
                            centerRow=5.0, centerCol=10.3, sod=30.0, sdd=70.0,
                            angles=[3.0, 47.5, 91.0, 150.2, 201.7, 266.0, 333.3])
    c["offset_parallel"] = dict(c["offset_cone"], geometry="parallel")
    del c["offset_parallel"]["sod"], c["offset_parallel"]["sdd"]
    c["offset_curved"] = dict(c["offset_cone"], geometry="cone-curved")
    # wide footprints near the source -> 2-way split path
    # (pkg/tests/test_sf.py:126-138)
    c["split_cone"] = dict(geometry="cone", numX=8, numY=8, numZ=4, voxelWidth=2.0,
                           voxelHeight=2.0, numRows=32, numCols=96, pixelHeight=1.0,
                           pixelWidth=0.5, sod=12.0, sdd=48.0, angles=[0.0, 45.0, 100.0])
    c["split_curved"] = dict(c["split_cone"], geometry="cone-curved")
    # source inside the grid: exercises the ok=False branches
    # (_kernels.py:468-469, 475-476, 511-520)
    c["inside_cone"] = dict(geometry="cone", numX=8, numY=8, numZ=3, voxelWidth=2.0,
                            voxelHeight=2.0, numRows=8, numCols=16, pixelHeight=2.0,
                            pixelWidth=2.0, sod=5.0, sdd=20.0,
                            angles=[0.0, 30.0, 90.0, 200.0])
    c["inside_curved"] = dict(c["inside_cone"], geometry="cone-curved")
    # fan beam = cone-flat with one row and one slice (gap 1)
    c["fan_like"] = dict(geometry="cone", numX=24, numY=24, numZ=1, voxelWidth=2.0,
                         voxelHeight=4.0, numRows=1, numCols=40, pixelHeight=1.0,
                         pixelWidth=1.5, sod=100.0, sdd=150.0,
                         angles=[360.0 * i / 16 for i in range(16)])
    # C3 optics (sod 1000 / sdd 1500, 0.6667 mm voxels, 1 mm pixels) on a
    # smaller grid, and C1 optics on a subset of its views
    c["c3_optics"] = dict(geometry="cone", numX=48, numY=48, numZ=40,
                          voxelWidth=0.6667, voxelHeight=0.6667,
                          numRows=72, numCols=72, pixelHeight=1.0, pixelWidth=1.0,
                          sod=1000.0, sdd=1500.0,
                          angles=[360.0 * i / 720 for i in (0, 37, 90, 181, 333, 600)])
    c["c1_views"] = dict(geometry="parallel", numX=128, numY=128, numZ=4,
                         voxelWidth=1.0, voxelHeight=1.0, numRows=4, numCols=128,
                         pixelHeight=1.0, pixelWidth=1.0,
                         angles=[180.0 * i / 180 for i in (0, 29, 45, 90, 133)])
    return c


def explicit_cases():
    # pkg/tests/test_sf.py:89-111
    base = dict(numX=5, numY=5, numZ=4, voxelWidth=1.0, voxelHeight=1.1,
                numRows=6, numCols=7, pixelHeight=1.3, pixelWidth=0.9,
                angles=[0.0, 60.0, 90.0, 145.0])
    return {
        "explicit_parallel": dict(base, geometry="parallel"),
        "explicit_cone": dict(base, geometry="cone", sod=18.0, sdd=36.0),
        "explicit_curved": dict(base, geometry="cone-curved", sod=18.0, sdd=36.0),
    }


def main():
    sys.path.insert(0, REF)
    import numba
    from ctproj import ProjectionSet, Volume, parse_config, sf_backproject, sf_forward

    numba.set_num_threads(min(8, numba.config.NUMBA_NUM_THREADS))
    blobs = {}
    for name, cfg in cases().items():
        g, spec = parse_config(json.dumps(cfg))
        rng_v = np.random.default_rng(0)
        rng_p = np.random.default_rng(1)
        x = rng_v.random(spec.shape, dtype=np.float32)
        y = rng_p.random(g.shape, dtype=np.float32)
        fx = sf_forward(Volume(spec, x), g).values
        by = sf_backproject(ProjectionSet(g, y), spec).values
        blobs[f"{name}.config"] = np.frombuffer(json.dumps(cfg).encode(), dtype=np.uint8)
        big = x.size > 40_000
        if big:
            # regenerate from the seed; store a checksum to detect RNG drift
            blobs[f"{name}.x_seed"] = np.array([0])
            blobs[f"{name}.x_sum"] = np.array([x.astype(np.float64).sum()])
        else:
            blobs[f"{name}.x"] = x
        blobs[f"{name}.y"] = y
        blobs[f"{name}.fwd"] = fx
        blobs[f"{name}.back"] = by
        print(name, spec.shape, g.shape, float(np.abs(fx).max()), float(np.abs(by).max()))
    for name, cfg in explicit_cases().items():
        g, spec = parse_config(json.dumps(cfg))
        n = int(np.prod(spec.shape))
        m = int(np.prod(g.shape))
        A = np.zeros((m, n), dtype=np.float32)
        for j in range(n):
            e = np.zeros(n, dtype=np.float32)
            e[j] = 1.0
            A[:, j] = sf_forward(Volume(spec, e.reshape(spec.shape)), g).values.ravel()
        B = np.zeros((n, m), dtype=np.float32)
        for i in range(m):
            e = np.zeros(m, dtype=np.float32)
            e[i] = 1.0
            B[:, i] = sf_backproject(ProjectionSet(g, e.reshape(g.shape)), spec).values.ravel()
        blobs[f"{name}.config"] = np.frombuffer(json.dumps(cfg).encode(), dtype=np.uint8)
        blobs[f"{name}.A"] = A
        blobs[f"{name}.B"] = B
        print(name, A.shape, float(np.abs(A - B.T).max()))
    np.savez_compressed(OUT, **blobs)
    print("wrote", OUT, os.path.getsize(OUT), "bytes")


if __name__ == "__main__":
    main()
