"""Device memory: the reference's memory criterion (7a) on the GPU and
streaming of problems larger than a device budget (north_star item 3).

Reference: pkg/tests/test_acceptance.py:265-290 (criterion 7a: peak extra
memory <= 1.25 x (volume + projection bytes) for forward and back
projection; "enough to hold one copy of the
projection data and volume data").  Here: peak extra device bytes of one
projector call on device-resident inputs (output + workspace), measured with
torch's allocator statistics, at C3 and the C2 fan batch.
"""

import json

import numpy as np
import pytest
import torch

import paper_2307_05801_b200 as ct
from paper_2307_05801_b200 import chunking, configs

from conftest import REARRANGE_TOL, rel_l2

pytestmark = pytest.mark.gpu

DEV = torch.device("cuda", 0)


def _pair(cfg):
    g, spec = ct.parse_config(json.dumps(cfg))
    return ct.ProjectorPair(ct.SF, g, spec)


def _peak_extra(fn):
    torch.cuda.synchronize()
    base = torch.cuda.memory_allocated(DEV)
    torch.cuda.reset_peak_memory_stats(DEV)
    out = fn()
    torch.cuda.synchronize()
    return torch.cuda.max_memory_allocated(DEV) - base, out


@pytest.mark.parametrize("which", ["c3", "c2"])
def test_memory_criterion_7a_on_device(which):
    cfg = configs.C3 if which == "c3" else configs.C2
    B = 1 if which == "c3" else configs.C2_BATCH
    P = _pair(cfg)
    plan = P.plan(0)
    vol_b = 4 * B * P.volumeSpec.num_voxels
    prj_b = 4 * B * int(np.prod(P.geometry.shape))
    x = torch.rand((B,) + P.volumeSpec.shape, device=DEV)
    y = torch.rand((B,) + P.geometry.shape, device=DEV)
    plan.forward(x)
    plan.back(y)  # plans and kernels warm
    budget = 1.25 * (vol_b + prj_b)
    fwd, yo = _peak_extra(lambda: plan.forward(x))
    del yo
    bwd, xo = _peak_extra(lambda: plan.back(y))
    del xo
    assert fwd <= budget and bwd <= budget, (fwd / budget, bwd / budget)


# a sinogram (11.1 MB) far above the cap: view chunks AND z-slabs
BIG = dict(geometry="cone", numX=48, numY=44, numZ=96, voxelWidth=0.8, voxelHeight=0.8,
           numRows=100, numCols=96, pixelHeight=1.0, pixelWidth=1.0, sod=400.0, sdd=600.0,
           numAngles=290, angularRange=360.0)


def test_streaming_within_device_budget(monkeypatch):
    P = _pair(BIG)
    g, spec = P.geometry, P.volumeSpec
    gen = np.random.default_rng(5)
    x = gen.random((1,) + spec.shape, dtype=np.float32)
    y = gen.random((1,) + g.shape, dtype=np.float32)
    ref_f = ct.forward(P, torch.from_numpy(x).to(DEV)).cpu().numpy()
    ref_b = ct.adjoint(P, torch.from_numpy(y).to(DEV)).cpu().numpy()
    budget = 1 << 20
    nzs, ranges = chunking.plan_blocks(g, spec, 1, budget)
    assert nzs < spec.numZ and len(ranges) > 1
    assert chunking.block_bytes(g, spec, 1, nzs, max(b - a for a, b in ranges)) <= budget
    monkeypatch.setenv("CTPROJ_DEVICE_BUDGET", str(budget))
    torch.cuda.synchronize()
    base = torch.cuda.memory_allocated(DEV)
    torch.cuda.reset_peak_memory_stats(DEV)
    got_f = ct.forward(P, x)
    got_b = ct.adjoint(P, y)
    peak = torch.cuda.max_memory_allocated(DEV) - base
    assert peak <= budget, (peak, budget)
    assert rel_l2(got_f, ref_f) < REARRANGE_TOL and rel_l2(got_b, ref_b) < REARRANGE_TOL


@pytest.mark.parametrize("direction", [0, 1])
@pytest.mark.parametrize("nzs,nvc,B", [(40, 7, 1), (17, 33, 2), (96, 290, 3)])
def test_stream_blocks_match_resident(direction, nzs, nvc, B):
    P = _pair(BIG)
    plan = P.plan(0)
    g, spec = P.geometry, P.volumeSpec
    shape = spec.shape if direction == 0 else g.shape
    h = torch.rand((B,) + shape)
    ref = (plan.forward if direction == 0 else plan.back)(h.to(DEV)).cpu()
    ranges = [(a, min(g.numViews, a + nvc)) for a in range(0, g.numViews, nvc)]
    got = chunking.stream_apply(plan, h, direction, nzs, ranges)
    assert rel_l2(got.numpy(), ref.numpy()) < REARRANGE_TOL
    if direction == 0 and nzs >= spec.numZ:
        assert torch.equal(got, ref)  # one slab: the same launches per view


def test_fan_batch_on_large_slices():
    """a 1600^2 slice (2.56M pixels) in the fan path needs more
    than 65535 transpose row blocks; it must run and agree with the
    per-element (3D kernel) path."""
    cfg = dict(geometry="cone", numX=1600, numY=1600, numZ=1, voxelWidth=0.25, voxelHeight=1.0,
               numRows=1, numCols=900, pixelHeight=1.0, pixelWidth=0.6, sod=1000.0, sdd=1500.0,
               numAngles=6, angularRange=360.0)
    P = _pair(cfg)
    x = torch.rand((2, 1, 1600, 1600), device=DEV)
    y = torch.rand((2,) + P.geometry.shape, device=DEV)
    fb, bb = ct.forward(P, x), ct.adjoint(P, y)
    for i in range(2):
        assert rel_l2(fb[i].cpu().numpy(), ct.forward(P, x[i:i + 1])[0].cpu().numpy()) < 1e-5
        assert rel_l2(bb[i].cpu().numpy(), ct.adjoint(P, y[i:i + 1])[0].cpu().numpy()) < 1e-5
