"""Shared fixtures.  Markers: ``gpu`` = needs a CUDA device (run on the B200
box with ``pytest -m gpu``); everything else runs on a CPU-only machine."""

import json
import os
import sys

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)

GOLDEN = os.path.join(ROOT, "tests", "golden", "sf_golden.npz")
SIDDON_GOLDEN = os.path.join(ROOT, "tests", "golden", "siddon_golden.npz")


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200)")


def load_golden(path=GOLDEN):
    z = np.load(path)
    cases = {}
    for key in z.files:
        name, field = key.split(".", 1)
        cases.setdefault(name, {})[field] = z[key]
    for name, c in cases.items():
        c["config"] = json.loads(bytes(c["config"]).decode())
        if "x" not in c and "x_seed" in c and "fwd" in c:
            from oracle import oracle

            vshape, _ = oracle.shapes(c["config"])
            c["x"] = np.random.default_rng(int(c["x_seed"][0])).random(vshape, dtype=np.float32)
    return cases


@pytest.fixture(scope="session")
def golden():
    return load_golden()


@pytest.fixture(scope="session")
def siddon_golden():
    return load_golden(SIDDON_GOLDEN)


@pytest.fixture(scope="session")
def oracle_mod():
    from oracle import oracle

    oracle.build()
    return oracle


def rel_l2(a, b):
    a = np.asarray(a, dtype=np.float64)
    b = np.asarray(b, dtype=np.float64)
    nb = np.linalg.norm(b)
    return float(np.linalg.norm(a - b) / nb) if nb > 0 else float(np.linalg.norm(a - b))


def max_abs_rel(a, b):
    a = np.asarray(a, dtype=np.float64)
    b = np.asarray(b, dtype=np.float64)
    m = float(np.abs(b).max())
    return float(np.abs(a - b).max() / m) if m > 0 else float(np.abs(a - b).max())


#: north_star tolerance: rel-L2 <= 1e-4 in fp32, stated max-abs bound 1e-4 * max|ref|
REL_L2_TOL = 1e-4
MAX_ABS_TOL = 1e-4
ADJOINT_TOL = 1e-5
# Two fp32 evaluations of the SAME projection under a different partition
# (z-slabs, view chunks, view shards, row sub-geometries): the integral
# formulation's prefix sums (csrc/sf_forward3d.cu, sf_back3d.cu) round
# differently per partition, ~1e-6 relative; 10x that, 10x inside the bar.
REARRANGE_TOL = 1e-5
#: explicit-matrix transpose bound of the 3D pair, relative to max|A| (fp32 rounding)
TRANSPOSE_TOL = 4e-6
