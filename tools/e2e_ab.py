"""Median wall time of host-buffer (e2e) forward / back calls on one config
(the path bench.py's e2e times); run under different CTPROJ_* settings to A/B
the host streaming.

    CTPROJ_FWD_STREAMS=1 python tools/e2e_ab.py --config c3 --n 7
"""
import argparse, json, os, statistics, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2307_05801_b200 as ct
from bench import CONFIGS

ap = argparse.ArgumentParser()
ap.add_argument("--config", default="c3")
ap.add_argument("--n", type=int, default=7)
a = ap.parse_args()
g, spec = ct.parse_config(json.dumps(CONFIGS[a.config]))
P = ct.ProjectorPair(ct.SF, g, spec)
xh = torch.rand((1,) + spec.shape).pin_memory()
yh = torch.rand((1,) + g.shape).pin_memory()
res = {"config": a.config, "env": {k: v for k, v in os.environ.items() if k.startswith("CTPROJ_")}}
outs = {}
for name, fn in (("forward", lambda: ct.forward(P, xh)), ("back", lambda: ct.adjoint(P, yh))):
    fn(); torch.cuda.synchronize()
    ms = []
    for _ in range(a.n):
        t0 = time.perf_counter()
        o = fn()
        torch.cuda.synchronize()
        ms.append((time.perf_counter() - t0) * 1e3)
    res[name + "_ms_median"] = round(statistics.median(ms), 2)
    res[name + "_ms"] = [round(m, 1) for m in ms]
    outs[name] = float(torch.as_tensor(o).double().sum())
res["sums"] = outs
print(json.dumps(res))
