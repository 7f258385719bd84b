"""SF-modular accuracy: the SF model on
modular poses has no reference counterpart (the reference raises for
SF + modular, pkg/src/ctproj/sf.py:23-27; its modular projector is Siddon,
_kernels.py:22-387), so it is pinned against the ANALYTIC projection of a
ball -- exact chord lengths, averaged over 3 x 3 rays per detector pixel --
on C4-like upright poses (source z +-50 mm, panel yaw +-5 deg, panel shift
+-20 mm), side by side with the GPU Siddon-modular pair, which is bitwise
equal to the reference (tests/test_gpu_siddon.py).  Tilted panels are
rejected (test_gpu_parity.py::test_sf_modular_rejects_tilted_panels)."""

import json

import numpy as np
import pytest
import torch

import paper_2307_05801_b200 as ct
from paper_2307_05801_b200 import configs

pytestmark = pytest.mark.gpu

N, H = 64, 2.0                  # 64^3 voxels of 2 mm
NR, NC, PW = 80, 96, 3.0        # detector rows x cols, 3 mm pixels
CEN, RAD = np.array([6.0, -4.0, 5.0]), 40.0


def _geometry(views, perturbed=True):
    """C4-like upright poses, or (perturbed=False) the plain cone orbit as
    modular poses -- the control SF models as well as cone-flat itself."""
    kw = {} if perturbed else dict(dz=0.0, rot_deg=0.0, shift=0.0)
    cfg = dict(geometry="modular", numX=N, numY=N, numZ=N, voxelWidth=H, voxelHeight=H,
               numRows=NR, numCols=NC, pixelHeight=PW, pixelWidth=PW,
               views=configs.modular_orbit(views, 1000.0, 1500.0, seed=11, tilt="yaw", **kw))
    return ct.parse_config(json.dumps(cfg))


def _ball_volume(ss=4):
    """Fractional occupancy of the ball per voxel (ss^3 sub-samples)."""
    c = (np.arange(N * ss) + 0.5) / ss * H - N * H / 2.0
    occ = np.zeros((N, N, N), np.float64)
    zz = c[:, None, None] - CEN[2]
    for iz in range(N):
        z = zz[iz * ss:(iz + 1) * ss]
        d2 = z ** 2 + (c[None, :, None] - CEN[1]) ** 2 + (c[None, None, :] - CEN[0]) ** 2
        inside = (d2 <= RAD * RAD).reshape(ss, N, ss, N, ss).mean(axis=(0, 2, 4))
        occ[iz] = inside
    return occ.astype(np.float32)


def _analytic(g, sub=3):
    """Chord lengths of the ball along source -> pixel rays, averaged over
    sub x sub rays per pixel (pixel centres: detectorCenter + (c - cc) pw u +
    (r - cr) ph v, the pose table of geometry.py)."""
    det = g.detector
    offs = (np.arange(sub) + 0.5) / sub - 0.5
    out = np.zeros((g.numViews, NR, NC))
    for k, mv in enumerate(g.modularViews):
        s = np.asarray(mv.sourcePos, float)
        acc = np.zeros((NR, NC))
        for a in offs:
            for b in offs:
                cc = (np.arange(NC) - det.centerCol + b) * PW
                rr = (np.arange(NR) - det.centerRow + a) * PW
                p = (np.asarray(mv.detectorCenter, float)[None, None, :]
                     + cc[None, :, None] * np.asarray(mv.colDir, float)[None, None, :]
                     + rr[:, None, None] * np.asarray(mv.rowDir, float)[None, None, :])
                d = p - s
                d /= np.linalg.norm(d, axis=-1, keepdims=True)
                w = CEN - s
                t = (d * w).sum(-1)
                dist2 = (w * w).sum() - t * t
                acc += 2.0 * np.sqrt(np.maximum(RAD * RAD - dist2, 0.0))
        out[k] = acc / (sub * sub)
    return out


def _rel(a, b):
    return float(np.linalg.norm((a - b).ravel()) / np.linalg.norm(b.ravel()))


def test_sf_modular_matches_analytic_ball():
    x = torch.from_numpy(_ball_volume()).cuda()
    errs = {}
    for name, pert in (("perturbed", True), ("unperturbed_control", False)):
        g, spec = _geometry(36, pert)
        ref = _analytic(g)
        sf = ct.forward(ct.ProjectorPair(ct.SF, g, spec), x[None])[0].cpu().numpy()
        sd = ct.forward(ct.ProjectorPair(ct.SIDDON, g, spec), x[None])[0].cpu().numpy()
        errs[name] = {"sf_modular_rel_rmse": _rel(sf, ref), "siddon_modular_rel_rmse": _rel(sd, ref)}
    print(json.dumps(errs))
    e_sf = errs["perturbed"]["sf_modular_rel_rmse"]
    e_sd = errs["perturbed"]["siddon_modular_rel_rmse"]
    e_ctrl = errs["unperturbed_control"]["sf_modular_rel_rmse"]
    # measured (B200): perturbed SF 1.20% / Siddon 2.26%; control 0.88% / 1.27%.
    # The perturbation makes the rays more oblique for BOTH models; the SF
    # footprint (exact for upright panels: the axial map stays affine in z)
    # keeps its lead over the reference's modular model (Siddon, one ray per
    # pixel) and does not lose accuracy relative to it.
    assert e_sf < 0.015, errs
    assert e_sf <= 0.75 * e_sd, errs
    ctrl_ratio = e_ctrl / errs["unperturbed_control"]["siddon_modular_rel_rmse"]
    assert e_sf / e_sd <= ctrl_ratio + 0.1, errs
