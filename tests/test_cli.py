"""CLI verbs (reference pkg/src/ctproj/cli.py): usage
and error exit codes on the CPU, every projector verb on the GPU against the
in-process public API, files in the reference's raw f32le + JSON format."""

import json

import numpy as np
import pytest
import torch

import paper_2307_05801_b200 as ct
from paper_2307_05801_b200 import cli

from conftest import rel_l2

CFG = dict(geometry="parallel", numX=24, numY=24, numZ=6, voxelWidth=1.0, voxelHeight=1.0,
           numRows=6, numCols=36, pixelHeight=1.0, pixelWidth=1.0, numAngles=30, angularRange=180.0)
CONE = dict(geometry="cone", numX=20, numY=20, numZ=12, voxelWidth=1.0, voxelHeight=1.0,
            numRows=16, numCols=32, pixelHeight=1.5, pixelWidth=1.5, sod=60.0, sdd=120.0, numAngles=24,
            angularRange=360.0)


def _write_cfg(tmp_path, cfg, name="cfg.json"):
    p = tmp_path / name
    p.write_text(json.dumps(cfg))
    return str(p)


def test_usage_errors_exit_2(capsys):
    for argv in ([], ["nonsense"], ["project", "--config", "c.json"], ["bench"]):
        with pytest.raises(SystemExit) as e:
            cli.main(argv)
        assert e.value.code == 2


def test_runtime_errors_exit_1(tmp_path, capsys):
    assert cli.main(["project", "--config", str(tmp_path / "missing.json"), "--in", "a", "--out", "b"]) == 1
    assert "error" in capsys.readouterr().err
    bad = tmp_path / "bad.json"
    bad.write_text("{not json")
    assert cli.main(["adjoint-check", "--config", str(bad)]) == 1


@pytest.mark.gpu
@pytest.mark.parametrize("cfg,model", [(CFG, "sf"), (CONE, "sf"), (CFG, "siddon")])
def test_project_backproject_match_api(tmp_path, capsys, cfg, model):
    cpath = _write_cfg(tmp_path, cfg)
    g, spec = ct.parse_config(json.dumps(cfg))
    P = ct.ProjectorPair(model, g, spec)
    rng = np.random.default_rng(3)
    x = ct.Volume(spec, rng.random(spec.shape, dtype=np.float32))
    y = ct.ProjectionSet(g, rng.random(g.shape, dtype=np.float32))
    ct.write_array(x, tmp_path / "x.json")
    ct.write_array(y, tmp_path / "y.json")
    assert cli.main(["project", "--config", cpath, "--model", model, "--in", str(tmp_path / "x.json"),
                     "--out", str(tmp_path / "Ax.json")]) == 0
    assert cli.main(["backproject", "--config", cpath, "--model", model, "--in", str(tmp_path / "y.json"),
                     "--out", str(tmp_path / "Aty.json")]) == 0
    out = capsys.readouterr().out.split()
    assert out == [str(tmp_path / "Ax.json"), str(tmp_path / "Aty.json")]
    np.testing.assert_array_equal(ct.read_array(tmp_path / "Ax.json").values, P.apply(x).values)
    np.testing.assert_array_equal(ct.read_array(tmp_path / "Aty.json").values, P.apply_adjoint(y).values)
    # a volume of the wrong spec is a runtime error (exit 1)
    bad = ct.Volume(ct.VolumeSpec(numX=4, numY=4, numZ=2, voxelWidth=1.0, voxelHeight=1.0),
                    np.zeros((2, 4, 4), np.float32))
    ct.write_array(bad, tmp_path / "bad.json")
    assert cli.main(["project", "--config", cpath, "--in", str(tmp_path / "bad.json"),
                     "--out", str(tmp_path / "o.json")]) == 1


@pytest.mark.gpu
def test_fbp_complete_refine_adjoint_bench(tmp_path, capsys):
    cpath = _write_cfg(tmp_path, CFG)
    g, spec = ct.parse_config(json.dumps(CFG))
    P = ct.ProjectorPair("sf", g, spec)
    rng = np.random.default_rng(4)
    x = ct.Volume(spec, rng.random(spec.shape, dtype=np.float32))
    y = P.apply(x)
    ct.write_array(x, tmp_path / "x.json")
    ct.write_array(y, tmp_path / "y.json")
    assert cli.main(["fbp", "--config", cpath, "--model", "sf", "--in", str(tmp_path / "y.json"),
                     "--out", str(tmp_path / "fbp.json")]) == 0
    ref = ct.fbp_parallel(y, spec, P).values
    assert rel_l2(ct.read_array(tmp_path / "fbp.json").values, ref) < 1e-6
    mask = [1 if i % 3 else 0 for i in range(g.numViews)]
    assert cli.main(["complete", "--config", cpath, "--model", "sf", "--in", str(tmp_path / "y.json"),
                     "--mask", json.dumps(mask), "--x0", str(tmp_path / "x.json"),
                     "--out", str(tmp_path / "c.json")]) == 0
    comp = ct.read_array(tmp_path / "c.json").values
    assert rel_l2(comp, y.values) < 1e-5  # x reproduces y, so the completed views agree
    assert cli.main(["refine", "--config", cpath, "--model", "sf", "--in", str(tmp_path / "y.json"),
                     "--mask", json.dumps(mask), "--x0", str(tmp_path / "x.json"), "--iters", "3",
                     "--out", str(tmp_path / "r.json")]) == 0
    assert cli.main(["recon-ls", "--config", cpath, "--model", "sf", "--in", str(tmp_path / "y.json"),
                     "--iters", "5", "--trace", str(tmp_path / "t.csv"), "--out", str(tmp_path / "ls.json")]) == 0
    assert open(tmp_path / "t.csv").readline().strip() == "iter,cost"
    capsys.readouterr()
    assert cli.main(["adjoint-check", "--config", cpath, "--model", "sf", "--trials", "3"]) == 0
    rep = json.loads(capsys.readouterr().out)
    assert rep["maxRelErr"] < 1e-5
    assert cli.main(["bench", "--config", cpath, "--model", "sf", "--repeat", "2"]) == 0
    b = json.loads(capsys.readouterr().out)
    assert b["model"] == "sf" and b["forward_median_s"] > 0 and b["backproject_median_s"] > 0
    assert b["volume_bytes"] == spec.num_voxels * 4 and b["projection_bytes"] == int(np.prod(g.shape)) * 4
