"""CPU-only tests of the host layer: config parsing, pose table / kernel
flattening vs the oracle's independent restatement, API contracts, and the
C-ABI library (loads, exports every declared symbol, validates arguments
without a GPU)."""

import ctypes
import json
import os
import re

import numpy as np
import pytest
import torch

import paper_2307_05801_b200 as ct
from paper_2307_05801_b200 import _native, errors
from paper_2307_05801_b200.ctproj_torch import NonContiguousError, Projector, ShapeMismatchError
from paper_2307_05801_b200.geometry import kernel_args

from conftest import ROOT, load_golden

HEADER = os.path.join(ROOT, "include", "ctproj_b200.h")


# ---------------------------------------------------------------------------
# configuration (geometry.py:431-512 semantics)
# ---------------------------------------------------------------------------
BASE = dict(geometry="cone", numRows=8, numCols=10, pixelHeight=1.0, pixelWidth=1.0,
            numX=6, numY=6, numZ=4, voxelWidth=1.0, voxelHeight=1.0, sod=50.0, sdd=100.0,
            numAngles=12, angularRange=360.0)


def test_parse_roundtrip():
    g, spec = ct.parse_config(json.dumps(BASE))
    assert g.kind == ct.CONE_FLAT and g.shape == (12, 8, 10) and spec.shape == (4, 6, 6)
    assert g.angles[1] == pytest.approx(30.0)
    g2, spec2 = ct.parse_config(ct.config_text(g, spec))
    assert g2 == g and spec2 == spec


@pytest.mark.parametrize("mutate,exc", [
    (lambda d: d.update(numAngels=3), errors.UnknownKeyError),
    (lambda d: d.pop("numRows"), errors.MissingKeyError),
    (lambda d: d.update(numRows=2.5), errors.InvalidValueError),
    (lambda d: d.update(angles=[0.0, 1.0]), errors.ConflictingKeysError),
    (lambda d: d.update(geometry="fan"), errors.InvalidValueError),
    (lambda d: d.update(sod=200.0), errors.InvalidValueError),
    (lambda d: d.update(voxelWidth=0), errors.InvalidValueError),
    (lambda d: d.update(angularRange=-1.0), errors.InvalidValueError),
])
def test_parse_errors(mutate, exc):
    d = dict(BASE)
    mutate(d)
    with pytest.raises(exc):
        ct.parse_config(json.dumps(d))


def test_parallel_rejects_cone_keys():
    d = dict(BASE, geometry="parallel")
    with pytest.raises(errors.UnknownKeyError, match="sdd|sod"):
        ct.parse_config(json.dumps(d))


def test_error_hierarchy_matches_reference():
    for cls in (errors.ConfigError, errors.UnsupportedGeometryError, errors.SpecMismatchError):
        assert issubclass(cls, errors.CtprojError) and issubclass(cls, ValueError)
    assert issubclass(errors.UnknownKeyError, errors.ConfigError)


# ---------------------------------------------------------------------------
# pose table / flattening vs the oracle's independent restatement
# ---------------------------------------------------------------------------
@pytest.mark.parametrize("name", sorted(load_golden()))
def test_kernel_args_match_oracle(golden, oracle_mod, name):
    cfg = golden[name]["config"]
    g, spec = ct.parse_config(json.dumps(cfg))
    a = kernel_args(g, spec)
    og, keep = oracle_mod.flatten(cfg)
    np.testing.assert_array_equal(a["poses"].reshape(-1, 15), keep)
    for f in ("kind", "num_views", "num_rows", "num_cols", "num_x", "num_y", "num_z",
              "pixel_width", "pixel_height", "center_row", "center_col", "sdd", "x0", "y0",
              "z0", "voxel_width", "voxel_height"):
        assert a[f] == getattr(og, f), f


def test_to_modular_poses_equal_cone():
    g, spec = ct.parse_config(json.dumps(BASE))
    gm = ct.to_modular(g)
    for a, b in zip(ct.pose_table(g), ct.pose_table(gm)):
        np.testing.assert_allclose(a, b, atol=1e-12)
    with pytest.raises(errors.UnsupportedGeometryError):
        ct.to_modular(gm)


# ---------------------------------------------------------------------------
# operator / binding contracts (no device needed to reach the checks)
# ---------------------------------------------------------------------------
def _pair():
    g, spec = ct.parse_config(json.dumps(BASE))
    return ct.ProjectorPair(ct.SF, g, spec)


def test_pair_model_checks():
    g, spec = ct.parse_config(json.dumps(BASE))
    with pytest.raises(errors.SpecMismatchError):
        ct.ProjectorPair("fancy", g, spec)
    # SF-modular is an extension of this build; poses whose rows do not point
    # upward are rejected
    ct.ProjectorPair(ct.SF, ct.to_modular(g), spec)
    gm = ct.to_modular(g)
    flipped = tuple(ct.ModularView(mv.sourcePos, mv.detectorCenter, -mv.rowDir, mv.colDir)
                    for mv in gm.modularViews)
    with pytest.raises(errors.UnsupportedGeometryError):
        ct.ProjectorPair(ct.SF, ct.Geometry(kind=ct.MODULAR, detector=g.detector,
                                            modularViews=flipped), spec)
    # the Siddon pair exists for every kind, modular poses of any orientation included
    ct.ProjectorPair(ct.SIDDON, g, spec)
    ct.ProjectorPair(ct.SIDDON, ct.Geometry(kind=ct.MODULAR, detector=g.detector, modularViews=flipped), spec)


def test_apply_spec_mismatch():
    P = _pair()
    other = ct.VolumeSpec(numX=5, numY=6, numZ=4, voxelWidth=1.0, voxelHeight=1.0)
    with pytest.raises(errors.SpecMismatchError):
        P.apply(ct.Volume(other, np.zeros(other.shape, np.float32)))
    g2 = P.geometry.with_views([0, 1])
    with pytest.raises(errors.SpecMismatchError):
        P.apply_adjoint(ct.ProjectionSet(g2, np.zeros(g2.shape, np.float32)))


def test_batch_rank_checked():
    P = _pair()
    with pytest.raises(errors.SpecMismatchError):
        ct.forward(P, np.zeros(P.volumeSpec.shape, np.float32))


def test_containers_reject_nonfinite_and_size():
    spec = _pair().volumeSpec
    bad = np.zeros(spec.shape, np.float32)
    bad[0, 0, 0] = np.nan
    with pytest.raises(errors.NonFiniteDataError):
        ct.Volume(spec, bad)
    with pytest.raises(errors.SizeMismatchError):
        ct.Volume(spec, np.zeros(7, np.float32))


def test_binding_contracts(tmp_path):
    cfg = tmp_path / "cfg.json"
    cfg.write_text(json.dumps(BASE))
    from paper_2307_05801_b200.ctproj_torch import load_param

    proj = load_param(cfg)
    assert proj.volume_shape == (4, 6, 6) and proj.projection_shape == (12, 8, 10)
    with pytest.raises(ShapeMismatchError):
        proj(torch.zeros(1, 3, 3, 3))
    with pytest.raises(ShapeMismatchError):
        proj(torch.zeros(1, 4, 6, 6, dtype=torch.float64))
    with pytest.raises(ShapeMismatchError):
        proj(torch.zeros(2, 4, 6, 6))
    big = torch.zeros(1, 4, 6, 12)
    with pytest.raises(NonContiguousError):
        proj(big[..., ::2])
    with pytest.raises(ShapeMismatchError):
        Projector()(torch.zeros(1, 2, 2, 2))
    bad = tmp_path / "bad.json"
    bad.write_text(json.dumps({"geometry": "parallel", "numAngels": 4}))
    with pytest.raises(errors.UnknownKeyError, match="numAngels"):
        load_param(bad)


@pytest.mark.skipif(torch.cuda.is_available(), reason="checks the no-GPU behaviour")
def test_no_silent_cpu_fallback():
    P = _pair()
    with pytest.raises((errors.CudaRuntimeError, errors.NativeLibraryError)):
        ct.forward(P, np.zeros((1,) + P.volumeSpec.shape, np.float32))


# ---------------------------------------------------------------------------
# C-ABI library
# ---------------------------------------------------------------------------
def _declared_functions():
    text = open(HEADER).read()
    return sorted(set(re.findall(r"^\s*(?:int|size_t|const char\*)\s+(ctp_\w+)\s*\(", text, re.M)))


def test_c4_pose_generator_is_seeded_and_valid():
    from paper_2307_05801_b200 import configs

    a, b = configs.c4(12, seed=3), configs.c4(12, seed=3)
    assert a == b
    g, spec = ct.parse_config(json.dumps(a))
    assert g.kind == ct.MODULAR and g.shape == (12, 384, 384) and spec.shape == (256, 256, 256)
    for mv in g.modularViews:
        assert mv.rowDir[2] > 0.99


def test_header_declarations_match_binding_list():
    assert _declared_functions() == sorted(_native.EXPORTED_SYMBOLS)


def test_library_exports_every_declared_symbol():
    lib = ctypes.CDLL(_native.LIB_PATH)
    for name in _declared_functions():
        assert hasattr(lib, name), name
    lib = _native.load_library()
    assert lib.ctp_abi_version() == _native.ABI_VERSION
    assert lib.ctp_status_string(2) == b"unsupported geometry"


def test_capi_validates_before_touching_the_device():
    lib = _native.load_library()
    h = ctypes.c_void_p()
    assert lib.ctp_plan_create(None, -1, ctypes.byref(h)) == 1
    g, spec = ct.parse_config(json.dumps(BASE))
    geom, keep = _native.make_geom(g, spec)
    geom.num_views = 0
    assert lib.ctp_plan_create(ctypes.byref(geom), -1, ctypes.byref(h)) == 1
    buf = ctypes.create_string_buffer(256)
    lib.ctp_last_error(buf, 256)
    assert b"counts" in buf.value
    # forward with a null plan is rejected, not crashed
    assert lib.ctp_sf_forward(None, None, None, 1, None, 0, 0, None) == 1
    assert lib.ctp_sf_workspace_bytes(None, 0, 1) == 0
    # the Siddon entry points validate the same way
    assert lib.ctp_siddon_forward(None, 1.0, None, None, 1, 0, None) == 1
    assert lib.ctp_siddon_back(None, 1.0, None, None, 1, 0, None) == 1


def test_stream_planner_respects_budget():
    """chunking.plan_blocks: view chunks, then z-slabs, within the budget."""
    from paper_2307_05801_b200 import chunking

    g, spec = ct.parse_config(json.dumps(dict(
        geometry="cone", numX=512, numY=512, numZ=512, voxelWidth=0.6667, voxelHeight=0.6667,
        numRows=768, numCols=768, pixelHeight=1.0, pixelWidth=1.0, sod=1000.0, sdd=1500.0,
        numAngles=720, angularRange=360.0)))
    big = 64 << 30
    nzs, ranges = chunking.plan_blocks(g, spec, 1, big)
    assert nzs == 512 and len(ranges) <= chunking.MAX_CHUNKS + 1  # (32-view multiples round down)
    for budget in (1 << 30, 256 << 20, 40 << 20):
        nzs, ranges = chunking.plan_blocks(g, spec, 1, budget)
        nvc = max(b - a for a, b in ranges)
        assert chunking.block_bytes(g, spec, 1, nzs, nvc) <= budget
        assert ranges[0][0] == 0 and ranges[-1][1] == 720
        assert all(r1[1] == r2[0] for r1, r2 in zip(ranges, ranges[1:]))
    nzs, _ = chunking.plan_blocks(g, spec, 1, 40 << 20)
    assert nzs < 512  # the volume no longer fits: z-slabs
    with pytest.raises(ct.CudaRuntimeError):
        chunking.plan_blocks(g, spec, 1, 1 << 20)


def test_taper_splits_the_exposed_chunk():
    """chunking.taper: the back's first chunk / the forward's last chunk is
    split so only 32 views wait on their transfer; coverage is unchanged."""
    from paper_2307_05801_b200 import chunking

    r = chunking.view_chunks(720, 768 * 768 * 4, (720 * 768 * 768 * 4 + 3) // 4)
    back, fwd = chunking.taper(r, 1), chunking.taper(r, 0)
    assert back[0] == (0, 32) and back[1] == (32, r[0][1]) and back[2:] == r[1:]
    assert fwd[-1] == (r[-1][1] - 32, r[-1][1]) and fwd[:-2] == r[:-1]
    for rs in (back, fwd):
        assert rs[0][0] == 0 and rs[-1][1] == 720
        assert all(a[1] == b[0] and a[0] < a[1] for a, b in zip(rs, rs[1:]))
    assert chunking.taper([(0, 720)], 1) == [(0, 720)]          # one chunk: nothing exposed to split
    assert chunking.taper([(0, 40), (40, 80)], 1) == [(0, 40), (40, 80)]  # too small to split
