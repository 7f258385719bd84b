"""Timeline of one host-buffer (e2e) forward and back call on C3 (torch.profiler
/ CUPTI): per call, wall time, the busy time of the compute kernels and of the
H2D / D2H copies, and the idle gaps of the compute stream -- where the e2e
overhead over the device-resident kernels goes.

    python tools/e2e_timeline.py [--config c3]
"""
import argparse, json, os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from torch.profiler import ProfilerActivity, profile
import paper_2307_05801_b200 as ct
from bench import CONFIGS

ap = argparse.ArgumentParser()
ap.add_argument("--config", default="c3")
a = ap.parse_args()
g, spec = ct.parse_config(json.dumps(CONFIGS[a.config]))
P = ct.ProjectorPair(ct.SF, g, spec)
xh = torch.rand((1,) + spec.shape).pin_memory()
yh = torch.rand((1,) + g.shape).pin_memory()
for _ in range(2):
    ct.forward(P, xh); ct.adjoint(P, yh)
torch.cuda.synchronize()
res = {}
for name, fn in (("forward", lambda: ct.forward(P, xh)), ("back", lambda: ct.adjoint(P, yh))):
    with profile(activities=[ProfilerActivity.CUDA, ProfilerActivity.CPU]) as prof:
        t0 = time.perf_counter()
        fn()
        torch.cuda.synchronize()
        wall = (time.perf_counter() - t0) * 1e3
    ev = [e for e in prof.events() if e.device_type == torch.autograd.DeviceType.CUDA]
    kern = [(e.time_range.start, e.time_range.end, e.name) for e in ev if "Memcpy" not in e.name and "Memset" not in e.name]
    h2d = [(e.time_range.start, e.time_range.end) for e in ev if "HtoD" in e.name]
    d2h = [(e.time_range.start, e.time_range.end) for e in ev if "DtoH" in e.name]
    allt = [t for s in (kern, h2d, d2h) for x in s for t in x[:2]]
    t_0 = min(allt)
    span = (max(allt) - t_0) / 1e3
    k = sorted(kern)
    per = {}
    for s, e, n in k:
        key = n.split("(")[0].split("<")[0][-40:]
        per[key] = per.get(key, 0.0) + (e - s) / 1e3
    first_k = (k[0][0] - t_0) / 1e3 if k else 0.0
    last_k = (max(kk[1] for kk in k) - t_0) / 1e3 if k else 0.0
    res[name] = {"wall_ms": round(wall, 1), "gpu_span_ms": round(span, 1),
                 "kernels_ms": {n: round(v, 2) for n, v in sorted(per.items(), key=lambda kv: -kv[1])},
                 "h2d_ms": round(sum(e - s for s, e in h2d) / 1e3, 1), "d2h_ms": round(sum(e - s for s, e in d2h) / 1e3, 1),
                 "first_kernel_at_ms": round(first_k, 1), "last_kernel_end_ms": round(last_k, 1),
                 "n_h2d": len(h2d), "n_d2h": len(d2h), "n_kernels": len(k)}
print(json.dumps(res, indent=1))
