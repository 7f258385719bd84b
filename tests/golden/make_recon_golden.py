"""Golden fixtures for the SF pair's callers, produced by
running the REAL reference (ctproj, /root/reference/pkg/src) in the build
container:

    PYTHONDONTWRITEBYTECODE=1 NUMBA_CACHE_DIR=/tmp/numba_cache \
        python tests/golden/make_recon_golden.py

Writes tests/golden/recon_golden.npz and tests/golden/io_ref/{vol,proj}.{json,raw}
(written by the reference's own write_array, datamodel.py:107-143).
"""

from __future__ import annotations

import json
import os
import sys

import numpy as np

REF = "/root/reference/pkg/src"
HERE = os.path.dirname(os.path.abspath(__file__))

PAR = dict(geometry="parallel", numX=20, numY=20, numZ=3, voxelWidth=1.2, voxelHeight=1.2,
           numRows=3, numCols=28, pixelHeight=1.2, pixelWidth=1.0,
           angles=[180.0 * i / 30 for i in range(30)])
CONE = dict(geometry="cone", numX=10, numY=10, numZ=8, voxelWidth=1.5, voxelHeight=1.5,
            numRows=12, numCols=16, pixelHeight=2.0, pixelWidth=2.0, sod=40.0, sdd=80.0,
            angles=[360.0 * i / 12 for i in range(12)])


def main():
    sys.path.insert(0, REF)
    from ctproj import (SF, AngleMask, LsConfig, ProjectionSet, ProjectorPair, Volume,
                        complete_sinogram, fbp_parallel, parse_config, reconstruct_ls,
                        refine_data_consistency, write_array)
    from ctproj.recon import ramp_filter_rows

    out = {}
    g, spec = parse_config(json.dumps(PAR))
    P = ProjectorPair(SF, g, spec)
    rng = np.random.default_rng(5)
    yv = rng.random(g.shape, dtype=np.float32)
    out["ramp_in"] = yv
    out["ramp_out"] = ramp_filter_rows(yv.astype(np.float64), g.detector.pixelWidth)
    out["fbp"] = fbp_parallel(ProjectionSet(g, yv), spec, P).values
    # a disk phantom and its SF projections (for LS)
    yy, xx = np.mgrid[0:20, 0:20]
    disk = ((xx - 9.5) ** 2 + (yy - 9.5) ** 2 < 49).astype(np.float32)
    x_true = np.repeat(disk[None], 3, axis=0) * 0.02
    y_true = P.apply(Volume(spec, x_true)).values
    out["ls_y"] = y_true
    x_ls, tr = reconstruct_ls(ProjectionSet(g, y_true), P, LsConfig(maxIters=8, step=2e-3))
    out["ls_x_explicit"] = x_ls.values
    out["ls_trace_explicit"] = np.array(tr)
    x_auto, tr_auto = reconstruct_ls(ProjectionSet(g, y_true), P, LsConfig(maxIters=6))
    out["ls_x_auto"] = x_auto.values
    out["ls_trace_auto"] = np.array(tr_auto)
    # cone: complete + refine
    gc, specc = parse_config(json.dumps(CONE))
    Pc = ProjectorPair(SF, gc, specc)
    xc = rng.random(specc.shape, dtype=np.float32)
    ym = rng.random(gc.shape, dtype=np.float32)
    keep = np.array([i % 3 != 1 for i in range(gc.numViews)])
    out["cone_x"] = xc
    out["cone_ym"] = ym
    out["cone_keep"] = keep
    out["complete"] = complete_sinogram(Volume(specc, xc), ProjectionSet(gc, ym), AngleMask(keep), Pc).values
    out["refine"] = refine_data_consistency(Volume(specc, xc), ProjectionSet(gc, ym), AngleMask(keep), Pc,
                                            LsConfig(maxIters=4, step=1e-3)).values
    out["par_config"] = np.frombuffer(json.dumps(PAR).encode(), dtype=np.uint8)
    out["cone_config"] = np.frombuffer(json.dumps(CONE).encode(), dtype=np.uint8)
    np.savez_compressed(os.path.join(HERE, "recon_golden.npz"), **out)
    io_dir = os.path.join(HERE, "io_ref")
    os.makedirs(io_dir, exist_ok=True)
    write_array(Volume(spec, x_true), os.path.join(io_dir, "vol.json"))
    write_array(ProjectionSet(g, y_true), os.path.join(io_dir, "proj.json"))
    print("ok", {k: getattr(v, "shape", None) for k, v in out.items()})


if __name__ == "__main__":
    main()
