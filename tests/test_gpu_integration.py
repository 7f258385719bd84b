"""The reference-side binding INTEGRATION.md §2 shows, executed verbatim.

The python block of INTEGRATION.md §2 (a ctypes stub that replaces
sf_forward_kernel / sf_back_kernel in ctproj/sf.py:30-45 with
ctp_sf_forward_oneshot / ctp_sf_back_oneshot) is extracted from the document,
pointed at the in-tree library and called with kernel_geom-shaped arguments
(_common.py:8-39: kind, src, c0, u, vax, w, pw, ph, cr, cc, sdd, back, x0, y0,
z0, hx, hz), exactly as the patched sf.py would.  Outputs must match the
reference's goldens.
"""

import os
import re

import numpy as np
import pytest

from conftest import MAX_ABS_TOL, REL_L2_TOL, ROOT, max_abs_rel, rel_l2

pytestmark = pytest.mark.gpu


def _binding():
    text = open(os.path.join(ROOT, "INTEGRATION.md")).read()
    sec = text[text.index("## 2."):]
    code = re.search(r"```python\n(.*?)```", sec, re.S).group(1)
    lib = os.path.join(ROOT, "paper_2307_05801_b200", "csrc", "libctproj_b200.so")
    code = code.replace('"/path/to/paper_2307_05801_b200/csrc/libctproj_b200.so"', repr(lib))
    ns = {}
    exec(compile(code, "INTEGRATION.md#2", "exec"), ns)
    return ns


def _kernel_geom(cfg):
    """kernel_geom's tuple (_common.py:8-39) from the oracle's independent flattening."""
    from oracle import oracle

    g, P = oracle.flatten(cfg)
    P = P.reshape(-1, 5, 3)
    back = oracle.siddon_back_offset(cfg)
    return (g.kind, P[:, 0], P[:, 1], P[:, 2], P[:, 3], P[:, 4], g.pixel_width, g.pixel_height,
            g.center_row, g.center_col, g.sdd, back, g.x0, g.y0, g.z0, g.voxel_width, g.voxel_height)


@pytest.mark.parametrize("name", ["cone_small", "parallel_small", "curved_small", "offset_cone", "c3_optics"])
def test_integration_stub_oneshot_matches_reference(golden, name):
    ns = _binding()
    c = golden[name]
    args = _kernel_geom(c["config"])
    out = np.empty(c["fwd"].shape, dtype=np.float32)
    ns["sf_forward_b200"](np.ascontiguousarray(c["x"], dtype=np.float32), out, args)
    assert rel_l2(out, c["fwd"]) <= REL_L2_TOL and max_abs_rel(out, c["fwd"]) <= MAX_ABS_TOL
    vol = np.empty(c["back"].shape, dtype=np.float32)
    ns["sf_back_b200"](np.ascontiguousarray(c["y"], dtype=np.float32), vol, args)
    assert rel_l2(vol, c["back"]) <= REL_L2_TOL and max_abs_rel(vol, c["back"]) <= MAX_ABS_TOL
