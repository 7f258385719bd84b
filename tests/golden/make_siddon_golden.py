"""Generate golden Siddon fixtures by running the REAL reference package.

Run in the build container (where /root/reference exists):

    PYTHONDONTWRITEBYTECODE=1 NUMBA_CACHE_DIR=/tmp/numba_cache \
        python tests/golden/make_siddon_golden.py

It imports ``ctproj`` from /root/reference/pkg/src (numba, read-only), runs
``siddon_forward`` / ``siddon_backproject`` (pkg/src/ctproj/siddon.py:18-31)
on seeded inputs and writes ``tests/golden/siddon_golden.npz``.  Cases cover
every geometry kind (parallel, cone-flat, cone-curved, modular), offsets,
shifted detector centres, rays along voxel boundary planes (axis-aligned
views, pkg/tests/test_siddon.py:127-135) and rays missing the grid; the
``explicit_*`` cases store the explicit forward matrix A and back matrix B
(pkg/tests/test_siddon.py:110-157).  Nothing on the GPU box reads
/root/reference; tests only read the committed .npz.
"""

from __future__ import annotations

import json
import os
import sys

import numpy as np

REF = "/root/reference/pkg/src"
OUT = os.path.join(os.path.dirname(os.path.abspath(__file__)), "siddon_golden.npz")


def cases():
    c = {}
    base = dict(numX=12, numY=12, numZ=12, voxelWidth=1.25, voxelHeight=1.25)
    c["parallel_small"] = dict(base, geometry="parallel", numRows=16, numCols=16,
                               pixelHeight=1.25, pixelWidth=1.25,
                               angles=[180.0 * i / 8 for i in range(8)])
    c["cone_small"] = dict(base, geometry="cone", numRows=16, numCols=16,
                           pixelHeight=2.0, pixelWidth=2.0, sod=40.0, sdd=80.0,
                           angles=[360.0 * i / 8 for i in range(8)])
    c["curved_small"] = dict(c["cone_small"], geometry="cone-curved")
    c["offset_cone"] = dict(geometry="cone", numX=10, numY=14, numZ=6,
                            voxelWidth=1.0, voxelHeight=1.3,
                            offsetX=0.8, offsetY=-0.4, offsetZ=0.2,
                            numRows=12, numCols=20, pixelHeight=1.1, pixelWidth=0.9,
                            centerRow=5.0, centerCol=10.3, sod=30.0, sdd=70.0,
                            angles=[3.0, 47.5, 91.0, 150.2, 201.7, 266.0, 333.3])
    c["offset_parallel"] = dict(c["offset_cone"], geometry="parallel")
    del c["offset_parallel"]["sod"], c["offset_parallel"]["sdd"]
    c["offset_curved"] = dict(c["offset_cone"], geometry="cone-curved")
    # rays along voxel boundary planes (axis-aligned views, pixel = voxel pitch)
    c["aligned_parallel"] = dict(numX=6, numY=6, numZ=6, voxelWidth=1.0, voxelHeight=1.0,
                                 geometry="parallel", numRows=8, numCols=8,
                                 pixelHeight=1.0, pixelWidth=1.0,
                                 angles=[0.0, 45.0, 90.0, 180.0, 270.0])
    # detector partly off the grid: rays that miss
    c["miss_parallel"] = dict(numX=8, numY=8, numZ=4, voxelWidth=1.0, voxelHeight=1.0,
                              geometry="parallel", numRows=6, numCols=10,
                              pixelHeight=1.0, pixelWidth=1.0, centerCol=-2.0,
                              angles=[0.0, 33.0, 120.0])
    # source inside the grid (the back projector's degenerate-window branch)
    c["inside_cone"] = dict(geometry="cone", numX=8, numY=8, numZ=3, voxelWidth=2.0,
                            voxelHeight=2.0, numRows=8, numCols=16, pixelHeight=2.0,
                            pixelWidth=2.0, sod=5.0, sdd=20.0,
                            angles=[0.0, 30.0, 90.0, 200.0])
    c["c3_optics"] = dict(geometry="cone", numX=32, numY=32, numZ=24,
                          voxelWidth=0.6667, voxelHeight=0.6667,
                          numRows=48, numCols=48, pixelHeight=1.0, pixelWidth=1.0,
                          sod=1000.0, sdd=1500.0,
                          angles=[360.0 * i / 720 for i in (0, 37, 90, 181, 333, 600)])
    return c


def modular_cases():
    """Perturbed cone orbit (source z, detector in-plane rotation and shift):
    the reference's only projector for modular geometry is Siddon."""
    rng = np.random.default_rng(4)
    views = []
    sod, sdd = 40.0, 80.0
    for i in range(6):
        phi = np.radians(360.0 * i / 6 + 7.0)
        r = np.array([np.cos(phi), np.sin(phi), 0.0])
        u = np.array([-np.sin(phi), np.cos(phi), 0.0])
        v = np.array([0.0, 0.0, 1.0])
        rot = np.radians(rng.uniform(-5.0, 5.0))
        u2 = np.cos(rot) * u + np.sin(rot) * v
        v2 = -np.sin(rot) * u + np.cos(rot) * v
        src = sod * r + np.array([0.0, 0.0, rng.uniform(-3.0, 3.0)])
        det = -(sdd - sod) * r + rng.uniform(-2.0, 2.0) * u
        views.append(dict(sourcePos=src.tolist(), detectorCenter=det.tolist(),
                          rowDir=v2.tolist(), colDir=u2.tolist()))
    return {"modular_perturbed": dict(geometry="modular", numX=10, numY=10, numZ=8,
                                      voxelWidth=1.5, voxelHeight=1.5, numRows=14,
                                      numCols=16, pixelHeight=1.8, pixelWidth=1.8,
                                      views=views)}


def explicit_cases():
    # pkg/tests/test_siddon.py:127-157
    sq = dict(numX=5, numY=5, numZ=5, voxelWidth=1.0, voxelHeight=1.0, numRows=6, numCols=6,
              pixelHeight=1.5, pixelWidth=1.5, angles=[0.0, 90.0, 210.0], sod=20.0, sdd=40.0)
    return {
        "explicit_boundary_parallel": dict(numX=4, numY=4, numZ=3, voxelWidth=1.0, voxelHeight=1.0,
                                           geometry="parallel", numRows=5, numCols=5,
                                           pixelHeight=1.2, pixelWidth=1.2,
                                           angles=[0.0, 45.0, 90.0, 180.0, 270.0]),
        "explicit_cone": dict(sq, geometry="cone"),
        "explicit_curved": dict(sq, geometry="cone-curved"),
    }


def main():
    sys.path.insert(0, REF)
    import numba
    from ctproj import ProjectionSet, Volume, parse_config, siddon_backproject, siddon_forward

    numba.set_num_threads(min(8, numba.config.NUMBA_NUM_THREADS))
    blobs = {}
    allc = dict(cases())
    allc.update(modular_cases())
    for name, cfg in allc.items():
        g, spec = parse_config(json.dumps(cfg))
        x = np.random.default_rng(0).random(spec.shape, dtype=np.float32)
        y = np.random.default_rng(1).random(g.shape, dtype=np.float32)
        fx = siddon_forward(Volume(spec, x), g).values
        by = siddon_backproject(ProjectionSet(g, y), spec).values
        blobs[f"{name}.config"] = np.frombuffer(json.dumps(cfg).encode(), dtype=np.uint8)
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
            A[:, j] = siddon_forward(Volume(spec, e.reshape(spec.shape)), g).values.ravel()
        B = np.zeros((n, m), dtype=np.float32)
        for i in range(m):
            e = np.zeros(m, dtype=np.float32)
            e[i] = 1.0
            B[:, i] = siddon_backproject(ProjectionSet(g, e.reshape(g.shape)), spec).values.ravel()
        blobs[f"{name}.config"] = np.frombuffer(json.dumps(cfg).encode(), dtype=np.uint8)
        blobs[f"{name}.A"] = A
        blobs[f"{name}.B"] = B
        print(name, A.shape, float(np.abs(A - B.T).max()))
    np.savez_compressed(OUT, **blobs)
    print("wrote", OUT, os.path.getsize(OUT), "bytes")


if __name__ == "__main__":
    main()
