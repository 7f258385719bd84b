"""Small SF + Siddon runs (every golden geometry, batch 2) for compute-sanitizer."""
import json, os, sys
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))
import torch
import paper_2307_05801_b200 as ct
from conftest import GOLDEN, SIDDON_GOLDEN, load_golden
dev = torch.device("cuda", 0)
n = 0
for path, model in ((GOLDEN, ct.SF), (SIDDON_GOLDEN, ct.SIDDON)):
    for name, c in load_golden(path).items():
        if name.startswith("explicit") or name.startswith("c1") or name.startswith("c3"):
            continue
        g, spec = ct.parse_config(json.dumps(c["config"]))
        P = ct.ProjectorPair(model, g, spec)
        x = torch.rand((2,) + spec.shape, device=dev)
        y = torch.rand((2,) + g.shape, device=dev)
        ct.forward(P, x); ct.adjoint(P, y)
        n += 1
torch.cuda.synchronize()
print("ok", n)
