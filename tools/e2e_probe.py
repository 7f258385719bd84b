"""Break down the host-buffer (e2e) path of one C3 fwd+back step."""
import json, sys, time, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2307_05801_b200 as ct
from paper_2307_05801_b200 import configs, chunking

g, spec = ct.parse_config(json.dumps(configs.C3))
P = ct.ProjectorPair(ct.SF, g, spec)
dev = torch.device("cuda", 0)
x = torch.rand((1,) + spec.shape, device=dev)
y = torch.rand((1,) + g.shape, device=dev)
xh, yh = x.cpu().pin_memory(), y.cpu().pin_memory()
plan = P.plan(0)

def t(f, n=2):
    f(); torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(n): f()
    torch.cuda.synchronize()
    return (time.perf_counter() - t0) / n * 1e3

res = {}
res["dev_fwd_ms"] = t(lambda: plan.forward(x))
res["dev_back_ms"] = t(lambda: plan.back(y))
res["h2d_x_ms"] = t(lambda: xh.to(dev, non_blocking=True))
res["h2d_y_ms"] = t(lambda: yh.to(dev, non_blocking=True))
ob = torch.empty_like(yh).pin_memory()
res["d2h_y_ms"] = t(lambda: ob.copy_(y, non_blocking=True))
res["host_fwd_ms"] = t(lambda: chunking.host_apply(plan, xh, 0))
res["host_back_ms"] = t(lambda: chunking.host_apply(plan, yh, 1))
res["api_fwd_ms"] = t(lambda: ct.forward(P, xh))
res["api_back_ms"] = t(lambda: ct.adjoint(P, yh))
res["pin_alloc_ms"] = t(lambda: torch.empty(yh.shape, pin_memory=True))
print(json.dumps(res))

# the bench's loop shape: results held across calls (steady-state pinned pool)
import time as _t
yo = xo = None
for _ in range(2):
    yo = ct.forward(P, xh); xo = ct.adjoint(P, yh)
torch.cuda.synchronize()
calls = []
for _ in range(3):
    t0 = _t.perf_counter(); yo = ct.forward(P, xh); t1 = _t.perf_counter(); xo = ct.adjoint(P, yh); t2 = _t.perf_counter()
    calls.append((round((t1 - t0) * 1e3, 1), round((t2 - t1) * 1e3, 1)))
print(json.dumps({"held_calls_ms": calls}))
