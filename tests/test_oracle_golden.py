"""Pin the CPU oracle (oracle/sf_oracle.c) to the REAL reference.

tests/golden/sf_golden.npz was produced by running the reference package
``ctproj`` (numba, /root/reference/pkg/src) with tests/golden/make_golden.py.
The oracle is a float64 restatement with the reference's operation order, so
it must reproduce the stored f32 outputs essentially bit for bit.
"""

import numpy as np
import pytest

from conftest import load_golden

CASES = sorted(n for n in load_golden() if not n.startswith("explicit"))
EXPLICIT = sorted(n for n in load_golden() if n.startswith("explicit"))


@pytest.mark.parametrize("name", CASES)
def test_oracle_forward_matches_reference(golden, oracle_mod, name):
    c = golden[name]
    got = oracle_mod.sf_forward(c["config"], c["x"])
    assert got.shape == c["fwd"].shape
    np.testing.assert_array_equal(got, c["fwd"])


@pytest.mark.parametrize("name", CASES)
def test_oracle_back_matches_reference(golden, oracle_mod, name):
    c = golden[name]
    got = oracle_mod.sf_back(c["config"], c["y"])
    np.testing.assert_array_equal(got, c["back"])


@pytest.mark.parametrize("name", EXPLICIT)
def test_oracle_explicit_matrices(golden, oracle_mod, name):
    c = golden[name]
    cfg = c["config"]
    vshape, sshape = oracle_mod.shapes(cfg)
    n, m = int(np.prod(vshape)), int(np.prod(sshape))
    A = np.zeros((m, n), dtype=np.float32)
    for j in range(n):
        e = np.zeros(n, dtype=np.float32)
        e[j] = 1.0
        A[:, j] = oracle_mod.sf_forward(cfg, e).ravel()
    np.testing.assert_array_equal(A, c["A"])
    # transpose property of the reference pair (pkg/tests/test_sf.py:89-111)
    assert np.abs(c["A"].astype(np.float64) - c["B"].T.astype(np.float64)).max() <= 1e-9


def test_oracle_thread_count_invariance(golden, oracle_mod):
    c = golden["cone_small"]
    a = oracle_mod.sf_forward(c["config"], c["x"], threads=1)
    b = oracle_mod.sf_forward(c["config"], c["x"], threads=4)
    np.testing.assert_array_equal(a, b)
    a = oracle_mod.sf_back(c["config"], c["y"], threads=1)
    b = oracle_mod.sf_back(c["config"], c["y"], threads=3)
    np.testing.assert_array_equal(a, b)


def test_oracle_rejects_modular(oracle_mod):
    cfg = {"geometry": "modular", "views": []}
    with pytest.raises(ValueError):
        oracle_mod.sf_forward(cfg, np.zeros(1, np.float32))


# ---- Siddon pair (oracle/siddon_oracle.c) ----------------------------------
from conftest import SIDDON_GOLDEN  # noqa: E402

SIDDON = load_golden(SIDDON_GOLDEN)
S_CASES = sorted(n for n in SIDDON if not n.startswith("explicit"))


@pytest.mark.parametrize("name", S_CASES)
def test_oracle_siddon_matches_reference(siddon_golden, oracle_mod, name):
    c = siddon_golden[name]
    np.testing.assert_array_equal(oracle_mod.siddon_forward(c["config"], c["x"]), c["fwd"])
    np.testing.assert_array_equal(oracle_mod.siddon_back(c["config"], c["y"]), c["back"])
