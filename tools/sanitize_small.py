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
# the integral kernels' paths (bands, pieces, clamped rows, ragged sizes,
# long tables, partial z-blocks) and the fused FBP input stage
from test_gpu_integral_paths import CASES
for name, cfg in CASES.items():
    g, spec = ct.parse_config(json.dumps(cfg))
    P = ct.ProjectorPair(ct.SF, g, spec)
    x = torch.rand((2,) + spec.shape, device=dev)
    y = torch.rand((2,) + g.shape, device=dev)
    ct.forward(P, x); ct.adjoint(P, y)
    n += 1
cfg = dict(geometry="parallel", numX=16, numY=16, numZ=3, voxelWidth=1.0, voxelHeight=1.0, numRows=3,
           numCols=37, pixelHeight=1.0, pixelWidth=0.75, numAngles=9, angularRange=180.0)
g, spec = ct.parse_config(json.dumps(cfg))
P = ct.ProjectorPair(ct.SF, g, spec)
P.plan().fbp_back(torch.rand((1,) + g.shape, device=dev), 0.5)
n += 1
torch.cuda.synchronize()
print("ok", n)
