"""GPU parity of the SF pair against the reference (golden fixtures) and the
CPU oracle, through the C-ABI library.

Bars (north_star): rel-L2 <= 1e-4 and max-abs <= 1e-4 * max|ref| for forward
and back projections; adjoint dot-product test <= 1e-5 relative; explicit
fp32 matrices transposed to fp32 rounding: max|A - B^T| <= TRANSPOSE_TOL *
max|A| for the 3D pair (the cumulative-footprint kernels evaluate the same
coefficient through two different prefix tables), bitwise for the fan pair
(the fp32 analogues of pkg/tests/test_sf.py:89-111's 1e-9 bound).
"""

import json

import numpy as np
import pytest
import torch

import paper_2307_05801_b200 as ct
from paper_2307_05801_b200 import _native

from conftest import (ADJOINT_TOL, MAX_ABS_TOL, REARRANGE_TOL, REL_L2_TOL, TRANSPOSE_TOL, load_golden, max_abs_rel,
                      rel_l2)

pytestmark = pytest.mark.gpu

DEV = torch.device("cuda", 0)
CASES = sorted(n for n in load_golden() if not n.startswith("explicit"))
EXPLICIT = sorted(n for n in load_golden() if n.startswith("explicit"))


def pair_of(cfg):
    g, spec = ct.parse_config(json.dumps(cfg))
    return ct.ProjectorPair(ct.SF, g, spec)


def dev_fwd(P, x):
    return ct.forward(P, torch.as_tensor(x, device=DEV).reshape((-1,) + P.volumeSpec.shape))


def dev_back(P, y):
    return ct.adjoint(P, torch.as_tensor(y, device=DEV).reshape((-1,) + P.geometry.shape))


def test_native_library_is_loaded():
    lib = _native.load_library()
    assert lib.ctp_abi_version() == _native.ABI_VERSION


@pytest.mark.parametrize("name", CASES)
def test_forward_matches_reference(golden, name):
    c = golden[name]
    P = pair_of(c["config"])
    got = dev_fwd(P, c["x"])[0].cpu().numpy()
    assert rel_l2(got, c["fwd"]) <= REL_L2_TOL, rel_l2(got, c["fwd"])
    assert max_abs_rel(got, c["fwd"]) <= MAX_ABS_TOL, max_abs_rel(got, c["fwd"])


@pytest.mark.parametrize("name", CASES)
def test_back_matches_reference(golden, name):
    c = golden[name]
    P = pair_of(c["config"])
    got = dev_back(P, c["y"])[0].cpu().numpy()
    assert rel_l2(got, c["back"]) <= REL_L2_TOL, rel_l2(got, c["back"])
    assert max_abs_rel(got, c["back"]) <= MAX_ABS_TOL, max_abs_rel(got, c["back"])


@pytest.mark.parametrize("name", EXPLICIT)
def test_explicit_matrices_exact_transpose(golden, name):
    c = golden[name]
    P = pair_of(c["config"])
    n = P.volumeSpec.num_voxels
    m = int(np.prod(P.geometry.shape))
    A = dev_fwd(P, torch.eye(n, device=DEV)).reshape(n, m).T.cpu().numpy()
    B = dev_back(P, torch.eye(m, device=DEV)).reshape(m, n).T.cpu().numpy()
    # the fp32 pair is a transpose to fp32 rounding
    assert np.abs(A - B.T).max() <= TRANSPOSE_TOL * np.abs(A).max(), np.abs(A - B.T).max() / np.abs(A).max()
    # and matches the reference's f64-computed matrix to fp32 accuracy
    assert np.abs(A - c["A"]).max() <= 1e-5 * np.abs(c["A"]).max()


@pytest.mark.parametrize("name", ["parallel_small", "cone_small", "curved_small", "offset_cone",
                                  "split_cone", "fan_like"])
def test_adjoint_check(golden, name):
    P = pair_of(golden[name]["config"])
    rep = ct.adjoint_check(P, trials=5, seed=0)
    assert rep["maxRelErr"] < ADJOINT_TOL, rep


def test_batch_equals_separate_calls_and_is_deterministic(golden):
    c = golden["cone_small"]
    P = pair_of(c["config"])
    x = torch.rand((3,) + P.volumeSpec.shape, device=DEV)
    yb = ct.forward(P, x)
    for i in range(3):
        assert torch.equal(yb[i], ct.forward(P, x[i:i + 1])[0])
    assert torch.equal(yb, ct.forward(P, x))
    y = torch.rand((3,) + P.geometry.shape, device=DEV)
    xb = ct.adjoint(P, y)
    for i in range(3):
        assert torch.equal(xb[i], ct.adjoint(P, y[i:i + 1])[0])
    assert torch.equal(xb, ct.adjoint(P, y))


def test_host_path_matches_device_path(golden):
    c = golden["offset_cone"]
    P = pair_of(c["config"])
    x = c["x"][None]
    host = ct.forward(P, x)
    assert isinstance(host, np.ndarray)
    dev = dev_fwd(P, x).cpu().numpy()
    assert np.array_equal(host, dev)
    yh = ct.adjoint(P, c["y"][None])
    yd = dev_back(P, c["y"]).cpu().numpy()
    assert np.array_equal(yh, yd)


def test_chunked_host_path(golden):
    from paper_2307_05801_b200 import chunking

    c = golden["cone_small"]
    P = pair_of(c["config"])
    plan = P.plan(0)
    xh = torch.from_numpy(c["x"][None].copy())
    yh = torch.from_numpy(c["y"][None].copy())
    one = chunking.host_apply(plan, xh, 0)
    many = chunking.host_apply(plan, xh, 0, chunk_bytes=16 * 16 * 4 * 3)  # 3 views per chunk
    assert torch.equal(one, many)  # (chunks alternate on two compute streams, ring slots reused)
    streams, chunking.FWD_STREAMS = chunking.FWD_STREAMS, 1
    try:
        serial = chunking.host_apply(plan, xh, 0, chunk_bytes=16 * 16 * 4 * 3)
    finally:
        chunking.FWD_STREAMS = streams
    assert torch.equal(serial, many)
    b1 = chunking.host_apply(plan, yh, 1)
    b3 = chunking.host_apply(plan, yh, 1, chunk_bytes=16 * 16 * 4 * 3)
    assert rel_l2(b3.numpy(), b1.numpy()) < REARRANGE_TOL


def test_binding_autograd_is_native_adjoint_bitwise(golden, tmp_path):
    from paper_2307_05801_b200.ctproj_torch import load_param

    c = golden["parallel_small"]
    cfg = tmp_path / "cfg.json"
    cfg.write_text(json.dumps(c["config"]))
    proj = load_param(cfg, model=ct.SF)
    P = proj.pair
    x = torch.rand((1,) + P.volumeSpec.shape, device=DEV, requires_grad=True)
    ybar = torch.rand((1,) + P.geometry.shape, device=DEV)
    y = proj(x)
    assert torch.equal(y, ct.forward(P, x.detach()))
    y.backward(ybar)
    assert torch.equal(x.grad, ct.adjoint(P, ybar))
    yy = torch.rand((1,) + P.geometry.shape, device=DEV, requires_grad=True)
    xx = proj.backproject(yy)
    xbar = torch.rand((1,) + P.volumeSpec.shape, device=DEV)
    xx.backward(xbar)
    assert torch.equal(yy.grad, ct.forward(P, xbar))
    # CPU tensors are accepted and give the same numbers
    xc = x.detach().cpu()
    assert torch.equal(proj(xc), y.detach().cpu())


def test_training_loop_decreases_loss(golden):
    from paper_2307_05801_b200.ctproj_torch import Projector

    c = golden["cone_small"]
    proj = Projector(pair_of(c["config"]))
    truth = torch.from_numpy(c["x"]).to(DEV)[None]
    with torch.no_grad():
        target = proj(truth)
    x = torch.zeros_like(truth, requires_grad=True)
    opt = torch.optim.SGD([x], lr=2e-4)
    losses = []
    for _ in range(30):
        opt.zero_grad()
        loss = 0.5 * ((proj(x) - target) ** 2).sum()
        loss.backward()
        opt.step()
        losses.append(loss.item())
    assert losses[-1] < 0.5 * losses[0]
    assert sum(b < a for a, b in zip(losses, losses[1:])) >= 27


# ---------------------------------------------------------------------------
# the BASELINE configs against the oracle (full geometry, view subsets)
# ---------------------------------------------------------------------------
C1 = dict(geometry="parallel", numX=128, numY=128, numZ=128, voxelWidth=1.0, voxelHeight=1.0,
          numRows=128, numCols=128, pixelHeight=1.0, pixelWidth=1.0, numAngles=180,
          angularRange=180.0)
C3 = dict(geometry="cone", numX=512, numY=512, numZ=512, voxelWidth=0.6667, voxelHeight=0.6667,
          numRows=768, numCols=768, pixelHeight=1.0, pixelWidth=1.0, sod=1000.0, sdd=1500.0,
          numAngles=720, angularRange=360.0)
C2 = dict(geometry="cone", numX=512, numY=512, numZ=1, voxelWidth=0.6667, voxelHeight=1.0,
          numRows=1, numCols=768, pixelHeight=1.0, pixelWidth=1.0, sod=1000.0, sdd=1500.0,
          numAngles=720, angularRange=360.0)


def _parity(oracle_mod, cfg, batch=1, views=None, max_abs=MAX_ABS_TOL):
    if views is not None:
        from oracle import oracle as o

        cfg = o.with_views(cfg, views)
    P = pair_of(cfg)
    rng = np.random.default_rng(0)
    x = rng.random((batch,) + P.volumeSpec.shape, dtype=np.float32)
    y = np.random.default_rng(1).random((batch,) + P.geometry.shape, dtype=np.float32)
    fx = dev_fwd(P, x).cpu().numpy()
    by = dev_back(P, y).cpu().numpy()
    for b in range(batch):
        rf = oracle_mod.sf_forward(cfg, x[b])
        rb = oracle_mod.sf_back(cfg, y[b])
        assert rel_l2(fx[b], rf) <= REL_L2_TOL and max_abs_rel(fx[b], rf) <= max_abs, \
            (rel_l2(fx[b], rf), max_abs_rel(fx[b], rf))
        assert rel_l2(by[b], rb) <= REL_L2_TOL and max_abs_rel(by[b], rb) <= max_abs, \
            (rel_l2(by[b], rb), max_abs_rel(by[b], rb))
    return P


def test_c1_parallel_full(oracle_mod):
    _parity(oracle_mod, C1)


def test_c3_cone_view_subset(oracle_mod):
    _parity(oracle_mod, C3, views=[0, 97, 181, 500])


def test_c2_fan_batch_subset(oracle_mod):
    _parity(oracle_mod, C2, batch=2, views=list(range(0, 720, 8)))


# ---------------------------------------------------------------------------
# fan beam with a batch: batch-on-lanes kernels (nz == nr == 1, batch >= 2)
# ---------------------------------------------------------------------------
FAN = dict(geometry="cone", numX=40, numY=36, numZ=1, voxelWidth=2.0, voxelHeight=4.0,
           numRows=1, numCols=70, pixelHeight=1.0, pixelWidth=1.5, sod=100.0, sdd=150.0,
           angles=[360.0 * i / 24 + 1.3 for i in range(24)])


@pytest.mark.parametrize("batch", [2, 40, 131])
def test_fan_batch_path_matches_per_element(batch):
    P = pair_of(FAN)
    x = torch.rand((batch,) + P.volumeSpec.shape, device=DEV)
    y = torch.rand((batch,) + P.geometry.shape, device=DEV)
    fb = ct.forward(P, x)       # batch-on-lanes path
    bb = ct.adjoint(P, y)
    for i in (0, batch // 2, batch - 1):
        f1 = ct.forward(P, x[i:i + 1])[0]  # batch 1: 3D path
        b1 = ct.adjoint(P, y[i:i + 1])[0]
        assert rel_l2(fb[i].cpu(), f1.cpu()) < 1e-6
        assert rel_l2(bb[i].cpu(), b1.cpu()) < 1e-6


def test_fan_batch_explicit_transpose():
    cfg = dict(FAN, numX=5, numY=5, numCols=7, angles=[0.0, 60.0, 90.0, 145.0])
    P = pair_of(cfg)
    n = P.volumeSpec.num_voxels
    m = int(np.prod(P.geometry.shape))
    A = dev_fwd(P, torch.eye(n, device=DEV)).reshape(n, m).T.cpu().numpy()
    B = dev_back(P, torch.eye(m, device=DEV)).reshape(m, n).T.cpu().numpy()
    assert np.array_equal(A, B.T), np.abs(A - B.T).max()


def test_fan_batch_against_oracle_and_golden(golden, oracle_mod):
    c = golden["fan_like"]
    P = pair_of(c["config"])
    xb = np.stack([c["x"]] * 5)
    yb = np.stack([c["y"]] * 5)
    fx = dev_fwd(P, xb).cpu().numpy()
    by = dev_back(P, yb).cpu().numpy()
    for i in range(5):
        assert rel_l2(fx[i], c["fwd"]) <= REL_L2_TOL and max_abs_rel(fx[i], c["fwd"]) <= MAX_ABS_TOL
        assert rel_l2(by[i], c["back"]) <= REL_L2_TOL and max_abs_rel(by[i], c["back"]) <= MAX_ABS_TOL


def test_c2_fan_batch40_subset(oracle_mod):
    _parity(oracle_mod, C2, batch=40, views=list(range(0, 720, 45)))


# ---------------------------------------------------------------------------
# SF-modular (extension: the reference has no SF for modular geometry)
# ---------------------------------------------------------------------------
@pytest.mark.parametrize("name", ["cone_small", "offset_cone", "c3_optics", "split_cone"])
def test_modular_of_cone_flat_equals_cone_flat(golden, name):
    c = golden[name]
    P = pair_of(c["config"])
    Pm = ct.ProjectorPair(ct.SF, ct.to_modular(P.geometry), P.volumeSpec)
    x = torch.from_numpy(c["x"]).to(DEV)[None]
    y = torch.from_numpy(c["y"]).to(DEV)[None]
    assert rel_l2(ct.forward(Pm, x).cpu(), ct.forward(P, x).cpu()) < 1e-5
    assert rel_l2(ct.adjoint(Pm, y).cpu(), ct.adjoint(P, y).cpu()) < 1e-5
    # and therefore matches the reference cone-flat outputs
    assert rel_l2(ct.forward(Pm, x)[0].cpu().numpy(), c["fwd"]) <= REL_L2_TOL


def _perturbed(n=6, views=10, seed=1):
    from paper_2307_05801_b200 import configs

    cfg = dict(geometry="modular", numX=n, numY=n, numZ=n - 1, voxelWidth=1.5, voxelHeight=1.4,
               numRows=9, numCols=11, pixelHeight=1.7, pixelWidth=1.6,
               views=configs.modular_orbit(views, 40.0, 90.0, seed=seed, dz=4.0, rot_deg=5.0,
                                           shift=2.0, tilt="yaw"))
    return pair_of(cfg)


def test_modular_perturbed_exact_transpose():
    P = _perturbed()
    n = P.volumeSpec.num_voxels
    m = int(np.prod(P.geometry.shape))
    A = dev_fwd(P, torch.eye(n, device=DEV)).reshape(n, m).T.cpu().numpy()
    B = dev_back(P, torch.eye(m, device=DEV)).reshape(m, n).T.cpu().numpy()
    assert np.abs(A).sum() > 0
    assert np.abs(A - B.T).max() <= TRANSPOSE_TOL * np.abs(A).max(), np.abs(A - B.T).max() / np.abs(A).max()


def test_c4_modular_adjoint():
    from paper_2307_05801_b200 import configs

    P = pair_of(configs.c4_upright(360, seed=0))
    rep = ct.adjoint_check(P, trials=2, seed=0)
    assert rep["maxRelErr"] < ADJOINT_TOL, rep


def test_sf_modular_rejects_tilted_panels():
    from paper_2307_05801_b200 import configs

    g, spec = ct.parse_config(json.dumps(configs.c4(8, seed=0)))  # in-plane (roll) rotations
    with pytest.raises(ct.UnsupportedGeometryError):
        ct.ProjectorPair(ct.SF, g, spec)


def test_c5_cone_view_subset(oracle_mod):
    from paper_2307_05801_b200 import configs

    # 1536-row detector: positions are resolved relative to local origins from
    # an f64 axial map, so the standard max-abs bound holds on 8 views
    _parity(oracle_mod, configs.C5, views=[5, 183, 361, 539, 700, 901, 1080, 1300])


# tall voxel columns (512 slices: the back kernel's 16-slice lanes, both
# forward row bands) over 64 views (two 32-view setup blocks): C3 optics
TALL = dict(geometry="cone", numX=48, numY=40, numZ=512, voxelWidth=0.6667, voxelHeight=0.6667,
            numRows=768, numCols=96, pixelHeight=1.0, pixelWidth=1.0, sod=1000.0, sdd=1500.0,
            numAngles=64, angularRange=360.0)


def test_tall_columns_64_views(oracle_mod):
    _parity(oracle_mod, TALL)


def test_tall_columns_partial_block(oracle_mod):
    # nz = 300: the last slice block is partial, the forward's slices end mid-band
    _parity(oracle_mod, dict(TALL, numZ=300, numAngles=40, offsetZ=7.3))


def test_c3_full_against_fixture():
    """Full C3 (512^3, 720 views, 768^2) against sampled oracle outputs
    (tests/golden/make_c3_fixture.py)."""
    import os

    from paper_2307_05801_b200 import configs

    path = os.path.join(os.path.dirname(__file__), "golden", "c3_full_samples.npz")
    z = np.load(path)
    P = pair_of(configs.C3)
    x = np.random.default_rng(0).random(P.volumeSpec.shape, dtype=np.float32)
    y = np.random.default_rng(1).random(P.geometry.shape, dtype=np.float32)
    fx = dev_fwd(P, x)[0]
    views = torch.as_tensor(z["fwd_views"].astype(np.int64), device=DEV)
    idx = torch.as_tensor(z["fwd_idx"].astype(np.int64), device=DEV)
    got = fx[views[:, None], idx[..., 0], idx[..., 1]].cpu().numpy()
    ref = z["fwd_val"]
    assert rel_l2(got, ref) <= REL_L2_TOL and max_abs_rel(got, ref) <= MAX_ABS_TOL, (rel_l2(got, ref), max_abs_rel(got, ref))
    vs = fx[views].double().sum(dim=(1, 2)).cpu().numpy()
    assert np.abs(vs - z["fwd_view_sums"]).max() <= 1e-5 * np.abs(z["fwd_view_sums"]).max()
    del fx
    bx = dev_back(P, y)[0]
    bi = torch.as_tensor(z["back_idx"].astype(np.int64), device=DEV)
    got = bx[bi[:, 0], bi[:, 1], bi[:, 2]].cpu().numpy()
    ref = z["back_val"]
    assert rel_l2(got, ref) <= REL_L2_TOL and max_abs_rel(got, ref) <= MAX_ABS_TOL, (rel_l2(got, ref), max_abs_rel(got, ref))
    ss = bx.double().sum(dim=(1, 2)).cpu().numpy()
    assert np.abs(ss - z["back_slice_sums"]).max() <= 1e-5 * np.abs(z["back_slice_sums"]).max()
    assert abs(float(bx.double().sum()) - float(z["back_total"][0])) <= 1e-6 * float(z["back_total"][0])


@pytest.mark.parametrize("nzs", [5, 16])
def test_zslab_streaming_matches_resident(golden, nzs):
    from paper_2307_05801_b200 import chunking

    c = golden["c3_optics"]  # 48 x 48 x 40 grid, C3 optics
    P = pair_of(c["config"])
    plan = P.plan(0)
    xh = torch.from_numpy(c["x"][None].copy())
    yh = torch.from_numpy(c["y"][None].copy())
    f_slab = chunking.zslab_apply(plan, xh, 0, nzs)
    b_slab = chunking.zslab_apply(plan, yh, 1, nzs)
    f_ref = ct.forward(P, xh.to(DEV)).cpu()
    b_ref = ct.adjoint(P, yh.to(DEV)).cpu()
    assert rel_l2(f_slab.numpy(), f_ref.numpy()) < REARRANGE_TOL
    assert rel_l2(b_slab.numpy(), b_ref.numpy()) < REARRANGE_TOL
    assert rel_l2(f_slab[0].numpy(), c["fwd"]) <= REL_L2_TOL


def test_zslab_env_forces_streaming(golden, monkeypatch):
    c = golden["cone_small"]
    P = pair_of(c["config"])
    ref = ct.forward(P, c["x"][None])
    monkeypatch.setenv("CTPROJ_ZSLAB", "5")
    got = ct.forward(P, c["x"][None])
    assert rel_l2(got, ref) < REARRANGE_TOL


@pytest.mark.parametrize("world", [2, 4, 8])
def test_zslab_parallel_partition_on_device(world, oracle_mod):
    """Parallel beam, z-partitioned (partition.ZSlabParallelProjector): every
    rank's sub-problem run on this GPU; the row / slice pieces reassemble
    the single-GPU pair (fp32 offsets only) and the C1-style oracle."""
    from paper_2307_05801_b200 import partition

    cfg = dict(geometry="parallel", numX=64, numY=64, numZ=48, voxelWidth=1.0, voxelHeight=1.0,
               offsetZ=3.3, numRows=56, numCols=72, pixelHeight=1.0, pixelWidth=1.0,
               angles=[180.0 * i / 30 for i in range(30)])
    P = pair_of(cfg)
    rng = np.random.default_rng(7)
    x = torch.from_numpy(rng.random(P.volumeSpec.shape, dtype=np.float32))[None].to(DEV)
    y = torch.from_numpy(rng.random(P.geometry.shape, dtype=np.float32))[None].to(DEV)
    full_f = ct.forward(P, x)[0]
    full_b = ct.adjoint(P, y)[0]
    parts = [partition.ZSlabParallelProjector(P, r, world, device=DEV) for r in range(world)]
    fwd = torch.cat([zp.forward(x)[0] for zp in parts], dim=1)
    back = torch.cat([zp.back(y)[0] for zp in parts], dim=0)
    assert rel_l2(fwd.cpu().numpy(), full_f.cpu().numpy()) <= REARRANGE_TOL
    assert rel_l2(back.cpu().numpy(), full_b.cpu().numpy()) <= REARRANGE_TOL
    ref_f = oracle_mod.sf_forward(cfg, x[0].cpu().numpy())
    assert rel_l2(fwd.cpu().numpy(), ref_f) <= REL_L2_TOL
    assert max_abs_rel(fwd.cpu().numpy(), ref_f) <= MAX_ABS_TOL


# ---------------------------------------------------------------------------
# full BASELINE sizes: size-independent properties (the oracle is too slow
# for whole C3 / C5 projections; view subsets above pin the values)
# ---------------------------------------------------------------------------
@pytest.mark.parametrize("which", ["c3", "c5"])
def test_full_size_adjoint_and_linearity(which):
    """Whole C3 (512^3 x 720, 768^2) and C5 (1024^3 x 1440, 1536^2): the
    adjoint identity <Ax, y> = <x, A^T y> with U[0,1) inputs (no cancellation,
    north_star bar 1e-5), linearity A(x1 + x2) = A x1 + A x2 to fp32 rounding
    of the integral formulation's prefix sums,
    and run-to-run determinism of both directions."""
    from paper_2307_05801_b200 import configs

    cfg = configs.C3 if which == "c3" else configs.C5
    g, spec = ct.parse_config(json.dumps(cfg))
    P = ct.ProjectorPair(ct.SF, g, spec)
    plan = P.plan(0)
    gen = torch.Generator(device=DEV)
    gen.manual_seed(0)
    x = torch.rand((1,) + spec.shape, device=DEV, generator=gen)
    y = torch.rand((1,) + g.shape, device=DEV, generator=gen)
    ax = plan.forward(x)
    aty = plan.back(y)
    lhs = float((ax.double() * y.double()).sum())
    rhs = float((x.double() * aty.double()).sum())
    assert abs(lhs - rhs) / abs(lhs) <= ADJOINT_TOL, (lhs, rhs)
    assert torch.equal(plan.forward(x), ax) and torch.equal(plan.back(y), aty)
    del aty
    x2 = torch.rand((1,) + spec.shape, device=DEV, generator=gen)
    a12 = plan.forward(x + x2)
    a2 = plan.forward(x2)
    err = float((a12.double() - ax.double() - a2.double()).norm() / a12.double().norm())
    # fp32 rounding of the staged prefix sums (sf_forward3d.cu): each row value
    # is a difference of two prefix values of up to ~512 slices, ~1e-5 relative
    # per (column, row) and ~1e-6 over a ray -- 100x inside the 1e-4 parity bar
    assert err <= 5e-6, err


@pytest.mark.parametrize("world", [2, 3, 6])
def test_view_sharded_partials_on_device(world, golden):
    """The N-rank view-sharded pair (partition.ViewShardedProjector with the
    CUDA backend), every rank's shard run on this GPU: forward shards
    concatenate to the single-GPU forward bitwise (views are independent),
    and the per-rank partial volumes sum to the single-GPU back projection
    (what the NCCL reduce-scatter computes) to fp32 reassociation."""
    from paper_2307_05801_b200 import partition

    c = golden["c3_optics"]
    P = pair_of(c["config"])
    nv = P.geometry.numViews
    if world > nv:
        pytest.skip("more ranks than views")
    x = torch.from_numpy(c["x"])[None].to(DEV)
    y = torch.from_numpy(c["y"])[None].to(DEV)
    full_f = ct.forward(P, x)
    full_b = ct.adjoint(P, y)
    parts_f, total_b = [], None
    for r in range(world):
        sp = partition.ViewShardedProjector(P, r, world, device=DEV)
        a, b = sp.views
        parts_f.append(sp.forward(x))
        part = sp._partial(y[:, a:b].contiguous())[:, : P.volumeSpec.numZ]
        total_b = part.clone() if total_b is None else total_b + part
    assert torch.equal(torch.cat(parts_f, dim=1), full_f)
    assert rel_l2(total_b.cpu().numpy(), full_b.cpu().numpy()) <= REARRANGE_TOL


def test_c3_optics_curved_detector_subset(oracle_mod):
    """C3 optics with a curved (cylindrical) detector on a 256^3 grid and a
    view subset: the atan2 column map of the curved kind at scale."""
    cfg = dict(C3, geometry="cone-curved", numX=256, numY=256, numZ=256, voxelWidth=1.3333,
               voxelHeight=1.3333, numRows=384, numCols=384, pixelHeight=2.0, pixelWidth=2.0)
    _parity(oracle_mod, cfg, views=[0, 133, 301, 577])


def test_c3_optics_offsets_and_shifted_detector(oracle_mod):
    """C3 optics with the grid off-centre and the detector centre shifted
    (rays enter the grid obliquely at the edges, partial row windows)."""
    cfg = dict(C3, numX=192, numY=160, numZ=128, voxelWidth=1.0, voxelHeight=1.2, offsetX=15.0,
               offsetY=-9.0, offsetZ=11.0, numRows=300, numCols=360, centerRow=140.3, centerCol=170.8)
    _parity(oracle_mod, cfg, views=[7, 95, 260, 640])
