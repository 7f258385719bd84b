"""Reproduce bench.py's sequence (device steps, then the host-buffer e2e loop)
and time the phases of each host call (synchronised), to find one-off costs."""
import json, os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2307_05801_b200 as ct
from paper_2307_05801_b200 import configs, partition

g, spec = ct.parse_config(json.dumps(configs.C3))
P = ct.ProjectorPair(ct.SF, g, spec)
dev = torch.device("cuda", 0)
sh = partition.ViewShardedProjector(P, 0, 1, device=dev)
plan = sh.shard.plan(0)
x = torch.rand((1,) + spec.shape, device=dev)
y = torch.rand((1,) + g.shape, device=dev)
so = torch.empty((1,) + g.shape, device=dev)
for _ in range(5):
    plan.forward(x, out=so, time_kernel=True)
    v = plan.back(y, time_kernel=True)
torch.cuda.synchronize()
xh, yh = x.cpu().pin_memory(), y.cpu().pin_memory()
out = {"steps": []}
for it in range(5):
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    yo = ct.forward(sh.shard, xh)
    t1 = time.perf_counter()
    xo = ct.adjoint(sh.shard, yh)
    t2 = time.perf_counter()
    out["steps"].append([round((t1 - t0) * 1e3, 1), round((t2 - t1) * 1e3, 1)])
    out.setdefault("mem", []).append(round(torch.cuda.memory_reserved() / 2**30, 2))
print(json.dumps(out))
