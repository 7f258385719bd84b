"""Every code path of the integral-formulation kernels (csrc/sf_forward3d.cu,
csrc/sf_back3d.cu) against the CPU oracle (oracle/sf_oracle.c, pinned to the
reference) at the north_star bars: the 768-row and 384-row forward bands,
staged ranges longer than one 512-slice piece (generic pieces), columns whose
rows need the clamped (unpadded) evaluation, nz and nr that are not
multiples of 4 (scalar loads / generic tables), partial z-blocks of the back
kernel (256- and 128-slice warps), batches, and the accumulate flag."""

import json

import numpy as np
import pytest
import torch

import paper_2307_05801_b200 as ct

from conftest import MAX_ABS_TOL, REL_L2_TOL, max_abs_rel, rel_l2

pytestmark = pytest.mark.gpu
DEV = torch.device("cuda", 0)


def _cone(nx, nz, nr, nc, hz, ph, views, sod=300.0, sdd=450.0, hx=1.0, pw=1.0):
    return dict(geometry="cone", numX=nx, numY=nx, numZ=nz, voxelWidth=hx, voxelHeight=hz,
                numRows=nr, numCols=nc, pixelHeight=ph, pixelWidth=pw, sod=sod, sdd=sdd,
                numAngles=views, angularRange=360.0)


CASES = {
    # 768-row band (nz <= 512, nr > 384), whole columns in one piece
    "band768": _cone(24, 300, 420, 40, 1.0, 1.0, 6),
    # 384-row bands (nz > 512) and staged ranges longer than 512 slices (hz << ph)
    "pieces": _cone(12, 700, 130, 24, 0.25, 1.0, 5),
    # nz, nr not multiples of 4: scalar x loads, generic S tables
    "ragged": _cone(20, 37, 43, 30, 1.0, 1.0, 7),
    # tall detector: long S tables (direct back path past 896 rows) and partial back z-blocks
    "tall": _cone(10, 520, 1000, 16, 2.0, 1.0, 4),
    # small magnification step (B < 0.8): clamped forward rows, 256-slice back warps
    "clamped": _cone(16, 260, 200, 24, 0.5, 1.0, 6),
}


def _pair(cfg):
    g, spec = ct.parse_config(json.dumps(cfg))
    return ct.ProjectorPair(ct.SF, g, spec)


@pytest.mark.parametrize("name", sorted(CASES))
def test_integral_paths_match_oracle(oracle_mod, name):
    cfg = CASES[name]
    P = _pair(cfg)
    rng = np.random.default_rng(11)
    x = rng.random(P.volumeSpec.shape, dtype=np.float32)
    y = rng.random(P.geometry.shape, dtype=np.float32)
    fx = ct.forward(P, torch.from_numpy(x)[None].to(DEV))[0].cpu().numpy()
    by = ct.adjoint(P, torch.from_numpy(y)[None].to(DEV))[0].cpu().numpy()
    rf = oracle_mod.sf_forward(cfg, x)
    rb = oracle_mod.sf_back(cfg, y)
    assert rel_l2(fx, rf) <= REL_L2_TOL and max_abs_rel(fx, rf) <= MAX_ABS_TOL, (rel_l2(fx, rf), max_abs_rel(fx, rf))
    assert rel_l2(by, rb) <= REL_L2_TOL and max_abs_rel(by, rb) <= MAX_ABS_TOL, (rel_l2(by, rb), max_abs_rel(by, rb))


@pytest.mark.parametrize("name", ["band768", "pieces"])
def test_integral_batch_and_accumulate(name):
    P = _pair(CASES[name])
    plan = P.plan(0)
    rng = np.random.default_rng(12)
    x = torch.from_numpy(rng.random((3,) + P.volumeSpec.shape, dtype=np.float32)).to(DEV)
    y = torch.from_numpy(rng.random((3,) + P.geometry.shape, dtype=np.float32)).to(DEV)
    fb, bb = plan.forward(x), plan.back(y)
    for i in range(3):
        assert torch.equal(plan.forward(x[i:i + 1])[0], fb[i])
        assert torch.equal(plan.back(y[i:i + 1])[0], bb[i])
    acc = fb.clone()
    plan.forward(x, out=acc, accumulate=True)
    assert rel_l2(acc.cpu().numpy(), (2 * fb).cpu().numpy()) < 1e-6
    accb = bb.clone()
    plan.back(y, out=accb, accumulate=True)
    assert rel_l2(accb.cpu().numpy(), (2 * bb).cpu().numpy()) < 1e-6
