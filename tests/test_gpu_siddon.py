"""GPU parity of the Siddon pair (csrc/siddon_kernels.cu) against the real
reference's outputs (tests/golden/siddon_golden.npz, made by
tests/golden/make_siddon_golden.py from pkg/src/ctproj/siddon.py).

The kernels restate the reference's float64 arithmetic in the same order
(no contraction), so the f32 outputs agree with the reference's to float64
rounding: the bar here is rel-L2 <= 1e-6 (the north-star bar is 1e-4) with
max-abs <= 1e-5 * max|ref|.  Explicit matrices: GPU A == reference A and
A ~ B^T (pkg/tests/test_siddon.py:110-157: 1e-10 in float64, i.e. the same
f32 values).
"""

import json

import numpy as np
import pytest
import torch

import paper_2307_05801_b200 as ct

from conftest import ADJOINT_TOL, SIDDON_GOLDEN, load_golden, max_abs_rel, rel_l2

pytestmark = pytest.mark.gpu

DEV = torch.device("cuda", 0)
NAMES = sorted(load_golden(SIDDON_GOLDEN))
CASES = [n for n in NAMES if not n.startswith("explicit")]
EXPLICIT = [n for n in NAMES if n.startswith("explicit")]


def pair_of(cfg):
    g, spec = ct.parse_config(json.dumps(cfg))
    return ct.ProjectorPair(ct.SIDDON, g, spec)


@pytest.mark.parametrize("name", CASES)
def test_siddon_forward_matches_reference(siddon_golden, name):
    c = siddon_golden[name]
    P = pair_of(c["config"])
    got = ct.forward(P, torch.from_numpy(c["x"])[None].to(DEV))[0].cpu().numpy()
    assert rel_l2(got, c["fwd"]) <= 1e-6, rel_l2(got, c["fwd"])
    assert max_abs_rel(got, c["fwd"]) <= 1e-5, max_abs_rel(got, c["fwd"])


@pytest.mark.parametrize("name", CASES)
def test_siddon_back_matches_reference(siddon_golden, name):
    c = siddon_golden[name]
    P = pair_of(c["config"])
    got = ct.adjoint(P, torch.from_numpy(c["y"])[None].to(DEV))[0].cpu().numpy()
    assert rel_l2(got, c["back"]) <= 1e-6, rel_l2(got, c["back"])
    assert max_abs_rel(got, c["back"]) <= 1e-5, max_abs_rel(got, c["back"])


@pytest.mark.parametrize("name", EXPLICIT)
def test_siddon_explicit_matrices(siddon_golden, name):
    c = siddon_golden[name]
    P = pair_of(c["config"])
    n, m = int(np.prod(P.volumeSpec.shape)), int(np.prod(P.geometry.shape))
    A = ct.forward(P, torch.eye(n, device=DEV).reshape((n,) + P.volumeSpec.shape)).reshape(n, m).T
    B = ct.adjoint(P, torch.eye(m, device=DEV).reshape((m,) + P.geometry.shape)).reshape(m, n).T
    A, B = A.cpu().numpy(), B.cpu().numpy()
    scale = np.abs(c["A"]).max()
    assert np.abs(A - c["A"]).max() <= 1e-6 * scale
    assert np.abs(B - c["B"]).max() <= 1e-6 * scale
    assert np.abs(A - B.T).max() <= 1e-6 * scale


@pytest.mark.parametrize("name", ["parallel_small", "cone_small", "curved_small", "modular_perturbed"])
def test_siddon_adjoint(siddon_golden, name):
    P = pair_of(siddon_golden[name]["config"])
    res = ct.adjoint_check(P, trials=3, seed=0)
    assert res["maxRelErr"] <= ADJOINT_TOL, res


def test_siddon_batch_and_host_paths(siddon_golden):
    c = siddon_golden["offset_cone"]
    P = pair_of(c["config"])
    x = torch.rand((3,) + P.volumeSpec.shape, device=DEV)
    y = torch.rand((3,) + P.geometry.shape, device=DEV)
    fb, bb = ct.forward(P, x), ct.adjoint(P, y)
    for i in range(3):
        assert torch.equal(fb[i], ct.forward(P, x[i:i + 1])[0])
        assert torch.equal(bb[i], ct.adjoint(P, y[i:i + 1])[0])
    assert np.array_equal(ct.forward(P, x.cpu().numpy()), fb.cpu().numpy())  # host numpy path
    assert torch.equal(ct.adjoint(P, y.cpu()), bb.cpu())                      # CPU tensor path
    # the containers' apply / apply_adjoint and the module-level functions
    xv = ct.Volume(P.volumeSpec, c["x"])
    assert np.array_equal(P.apply(xv).values, ct.siddon_forward(xv, P.geometry).values)


def test_binding_default_model_is_siddon(siddon_golden, tmp_path):
    from paper_2307_05801_b200.ctproj_torch import load_param

    c = siddon_golden["cone_small"]
    cfg = tmp_path / "cfg.json"
    cfg.write_text(json.dumps(c["config"]))
    proj = load_param(cfg)  # reference default (TB:103)
    assert proj.pair.model == ct.SIDDON
    x = torch.from_numpy(c["x"])[None].to(DEV).requires_grad_(True)
    y = proj(x)
    assert rel_l2(y[0].detach().cpu().numpy(), c["fwd"]) <= 1e-6
    ybar = torch.rand_like(y)
    y.backward(ybar)
    assert torch.equal(x.grad, ct.adjoint(proj.pair, ybar))


@pytest.mark.parametrize("which", ["c1_parallel", "modular_c4_optics", "cone_curved"])
def test_siddon_against_oracle_at_scale(oracle_mod, which):
    """Larger grids than the goldens, against the C oracle (itself bitwise
    equal to the reference on every golden): C1 (parallel 128^3, 128^2) on a
    view subset, C4 optics (modular, perturbed poses) on a 96^3 grid, and a
    curved cone.  float64 without contraction on both sides: bitwise except
    for the curved detector (GPU vs glibc cos/sin/atan2)."""
    from paper_2307_05801_b200 import configs

    if which == "c1_parallel":
        cfg = dict(configs.C1)
        cfg.pop("numAngles"), cfg.pop("angularRange")
        cfg["angles"] = [180.0 * i / 180 for i in (0, 17, 45, 90, 121, 179)]
    elif which == "modular_c4_optics":
        c4 = configs.c4(n_views=6, seed=3)
        cfg = dict(c4, numX=96, numY=96, numZ=96, voxelWidth=3.5556, voxelHeight=3.5556,
                   numRows=144, numCols=144, pixelHeight=5.333, pixelWidth=5.333)
    else:
        cfg = dict(geometry="cone-curved", numX=64, numY=64, numZ=48, voxelWidth=1.0, voxelHeight=1.0,
                   numRows=64, numCols=96, pixelHeight=1.5, pixelWidth=1.5, sod=200.0, sdd=400.0,
                   angles=[0.0, 41.0, 133.0, 270.0])
    P = pair_of(cfg)
    rng = np.random.default_rng(11)
    x = rng.random(P.volumeSpec.shape, dtype=np.float32)
    y = rng.random(P.geometry.shape, dtype=np.float32)
    f = ct.forward(P, torch.from_numpy(x)[None].to(DEV))[0].cpu().numpy()
    b = ct.adjoint(P, torch.from_numpy(y)[None].to(DEV))[0].cpu().numpy()
    rf, rb = oracle_mod.siddon_forward(cfg, x), oracle_mod.siddon_back(cfg, y)
    if which == "cone_curved":
        assert rel_l2(f, rf) <= 1e-7 and rel_l2(b, rb) <= 1e-7
    else:
        np.testing.assert_array_equal(f, rf)
        np.testing.assert_array_equal(b, rb)
