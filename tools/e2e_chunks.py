"""Host-buffer (e2e) call times of the C3 pair vs the number of view chunks
(CTPROJ_MAX_CHUNKS / CTPROJ_CHUNK_BYTES are read at import: one process per
setting; run as `for m in 1 2 4 8; do CTPROJ_MAX_CHUNKS=$m CTPROJ_CHUNK_BYTES=1 python tools/e2e_chunks.py; done`)."""
import json, os, sys, time
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
for _ in range(2):
    yo = ct.forward(P, xh); xo = ct.adjoint(P, yh)
torch.cuda.synchronize()
calls = []
for _ in range(4):
    t0 = time.perf_counter(); yo = ct.forward(P, xh); t1 = time.perf_counter(); xo = ct.adjoint(P, yh)
    t2 = time.perf_counter()
    calls.append((round((t1 - t0) * 1e3, 1), round((t2 - t1) * 1e3, 1)))
nzs, ranges = chunking.plan_blocks(g, spec, 1, chunking.device_budget(dev))
print(json.dumps({"max_chunks": chunking.MAX_CHUNKS, "chunks": len(ranges), "nzs": nzs, "calls_ms": calls}))
