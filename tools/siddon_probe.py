"""Siddon pair on the GPU: parity against the committed reference goldens and
device timing (CUDA events) at C1 (parallel 128^3 x 180) and C4 (modular
256^3 x 360 perturbed poses, 384^2).  Prints one JSON object.

    python tools/siddon_probe.py
"""
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))

import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2307_05801_b200 as ct  # noqa: E402
from conftest import SIDDON_GOLDEN, load_golden, rel_l2  # noqa: E402
from paper_2307_05801_b200 import configs  # noqa: E402

dev = torch.device("cuda", 0)
out = {"parity": {}}
for name, c in load_golden(SIDDON_GOLDEN).items():
    if name.startswith("explicit"):
        continue
    g, spec = ct.parse_config(json.dumps(c["config"]))
    P = ct.ProjectorPair(ct.SIDDON, g, spec)
    f = ct.forward(P, torch.from_numpy(c["x"])[None].to(dev))[0].cpu().numpy()
    b = ct.adjoint(P, torch.from_numpy(c["y"])[None].to(dev))[0].cpu().numpy()
    out["parity"][name] = {"fwd_rel_l2": rel_l2(f, c["fwd"]), "back_rel_l2": rel_l2(b, c["back"]),
                           "fwd_bitwise_frac": float(np.mean(f == c["fwd"])),
                           "back_bitwise_frac": float(np.mean(b == c["back"]))}


def timed(plan, fn, inp, reps=3):
    fn(inp)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        fn(inp)
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps


for tag, cfg in (("c1", configs.C1), ("c4", configs.c4())):
    g, spec = ct.parse_config(json.dumps(cfg))
    P = ct.ProjectorPair(ct.SIDDON, g, spec)
    plan = P.plan(0)
    x = torch.rand((1,) + spec.shape, device=dev)
    y = torch.rand((1,) + g.shape, device=dev)
    tf = timed(plan, plan.siddon_forward, x)
    tb = timed(plan, plan.siddon_back, y)
    upd = spec.num_voxels * g.numViews
    adj = ct.adjoint_check(P, trials=1, seed=0)["maxRelErr"] if tag == "c4" else None
    out[tag] = {"fwd_ms": tf, "back_ms": tb, "gups_fwd_back": 2 * upd / ((tf + tb) / 1e3) / 1e9,
                "rays": int(np.prod(g.shape)), "voxels": spec.num_voxels, "views": g.numViews,
                "adjoint_rel": adj}
print(json.dumps(out))
