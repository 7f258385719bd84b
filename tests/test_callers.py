"""Callers of the SF pair against fixtures produced by the
real reference (tests/golden/make_recon_golden.py): raw+JSON array files
(CPU), ramp filter, FBP, least squares, sinogram completion and
data-consistency refinement (GPU)."""

import json
import os

import numpy as np
import pytest
import torch

import paper_2307_05801_b200 as ct
from paper_2307_05801_b200 import errors

from conftest import ROOT, rel_l2

GOLD = os.path.join(ROOT, "tests", "golden")


@pytest.fixture(scope="module")
def rg():
    z = np.load(os.path.join(GOLD, "recon_golden.npz"))
    d = {k: z[k] for k in z.files}
    d["par"] = ct.parse_config(bytes(d["par_config"]).decode())
    d["cone"] = ct.parse_config(bytes(d["cone_config"]).decode())
    return d


# ---------------------------------------------------------------------------
# f4: raw f32le + JSON header files (CPU)
# ---------------------------------------------------------------------------
def test_reads_files_written_by_the_reference(rg):
    g, spec = rg["par"]
    v = ct.read_array(os.path.join(GOLD, "io_ref", "vol.json"))
    p = ct.read_array(os.path.join(GOLD, "io_ref", "proj.json"))
    assert v.spec == spec and p.geometry == g
    np.testing.assert_array_equal(p.values, rg["ls_y"])


def test_write_matches_reference_bytes(rg, tmp_path):
    p = ct.read_array(os.path.join(GOLD, "io_ref", "proj.json"))
    ct.write_array(p, tmp_path / "proj.json")
    ref_raw = open(os.path.join(GOLD, "io_ref", "proj.raw"), "rb").read()
    assert open(tmp_path / "proj.raw", "rb").read() == ref_raw
    assert json.load(open(tmp_path / "proj.json")) == json.load(open(os.path.join(GOLD, "io_ref", "proj.json")))
    assert not any(f.endswith(".tmp") for f in os.listdir(tmp_path))


def test_read_errors(tmp_path):
    (tmp_path / "h.json").write_text("{not json")
    with pytest.raises(errors.MalformedHeaderError):
        ct.read_array(tmp_path / "h.json")
    (tmp_path / "s.json").write_text(json.dumps({"kind": "volume", "shape": [2, 2, 2], "dtype": "f32le",
                                                  "raw": "s.raw"}))
    (tmp_path / "s.raw").write_bytes(b"\0" * 12)
    with pytest.raises(errors.SizeMismatchError):
        ct.read_array(tmp_path / "s.json")


# ---------------------------------------------------------------------------
# f2 / f3 on the device
# ---------------------------------------------------------------------------
@pytest.mark.gpu
def test_ramp_filter(rg):
    g, _ = rg["par"]
    got = ct.ramp_filter_rows(rg["ramp_in"].astype(np.float64), g.detector.pixelWidth)
    assert rel_l2(got, rg["ramp_out"]) < 1e-12


@pytest.mark.gpu
def test_fbp_parallel(rg):
    g, spec = rg["par"]
    P = ct.ProjectorPair(ct.SF, g, spec)
    got = ct.fbp_parallel(ct.ProjectionSet(g, rg["ramp_in"]), spec, P).values
    assert isinstance(got, np.ndarray)
    assert rel_l2(got, rg["fbp"]) < 1e-5
    dev = ct.fbp_parallel(ct.ProjectionSet(g, torch.from_numpy(rg["ramp_in"]).cuda()), spec, P).values
    assert dev.is_cuda and rel_l2(dev.cpu().numpy(), rg["fbp"]) < 1e-5


@pytest.mark.gpu
@pytest.mark.parametrize("kind", ["explicit", "auto"])
def test_reconstruct_ls(rg, kind):
    g, spec = rg["par"]
    P = ct.ProjectorPair(ct.SF, g, spec)
    cfg = ct.LsConfig(maxIters=8, step=2e-3) if kind == "explicit" else ct.LsConfig(maxIters=6)
    x, trace = ct.reconstruct_ls(ct.ProjectionSet(g, rg["ls_y"]), P, cfg)
    ref_trace = rg[f"ls_trace_{kind}"]
    assert len(trace) == len(ref_trace)
    np.testing.assert_allclose(trace, ref_trace, rtol=1e-4)
    assert rel_l2(x.values, rg[f"ls_x_{kind}"]) < 1e-4


@pytest.mark.gpu
def test_complete_and_refine(rg):
    g, spec = rg["cone"]
    P = ct.ProjectorPair(ct.SF, g, spec)
    mask = ct.AngleMask(rg["cone_keep"])
    x = ct.Volume(spec, rg["cone_x"])
    ym = ct.ProjectionSet(g, rg["cone_ym"])
    comp = ct.complete_sinogram(x, ym, mask, P).values
    keep = rg["cone_keep"]
    np.testing.assert_array_equal(comp[keep], rg["complete"][keep])
    assert rel_l2(comp[~keep], rg["complete"][~keep]) < 1e-5
    ref = ct.refine_data_consistency(x, ym, mask, P, ct.LsConfig(maxIters=4, step=1e-3)).values
    assert rel_l2(ref, rg["refine"]) < 1e-5


@pytest.mark.gpu
def test_divergence_detected(rg):
    g, spec = rg["par"]
    P = ct.ProjectorPair(ct.SF, g, spec)
    with pytest.raises(errors.DivergenceDetectedError):
        ct.reconstruct_ls(ct.ProjectionSet(g, rg["ls_y"]), P, ct.LsConfig(maxIters=20, step=5.0))


def test_psnr():
    a = np.zeros(10)
    b = np.ones(10)
    assert ct.psnr(b, b) == float("inf")
    assert ct.psnr(a, b, peak=1.0) == pytest.approx(0.0)


@pytest.mark.gpu
@pytest.mark.parametrize("nc,nr", [(37, 5), (600, 3)])
def test_fused_ramp_back_matches_cufft_filter(nc, nr):
    """csrc/ramp_kernels.cu (direct linear convolution, fused with the back
    projection's input layout change) == cuFFT float64 ramp filter followed
    by the SF back projection, on detector rows that are not a multiple of 8
    and rows much wider than one tile."""
    cfg = dict(geometry="parallel", numX=16, numY=16, numZ=nr, voxelWidth=1.0, voxelHeight=1.0,
               numRows=nr, numCols=nc, pixelHeight=1.0, pixelWidth=0.75, numAngles=9, angularRange=180.0)
    g, spec = ct.parse_config(json.dumps(cfg))
    P = ct.ProjectorPair(ct.SF, g, spec)
    y = torch.from_numpy(np.random.default_rng(7).standard_normal(g.shape).astype(np.float32)).cuda()
    scale = 0.37
    got = P.plan().fbp_back(y[None], scale)[0]
    filt = ct.ramp_filter_rows(y.double(), g.detector.pixelWidth).float() * scale
    ref = P.plan().back(filt[None].contiguous())[0]
    assert rel_l2(got.cpu().numpy(), ref.cpu().numpy()) < 1e-5
