"""One Siddon back projection at C4 optics (modular 256^3, `views` poses) for profiling."""
import json, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2307_05801_b200 as ct
from paper_2307_05801_b200 import configs
views = int(sys.argv[1]) if len(sys.argv) > 1 else 36
g, spec = ct.parse_config(json.dumps(configs.c4(n_views=views)))
P = ct.ProjectorPair(ct.SIDDON, g, spec)
y = torch.rand((1,) + g.shape, device="cuda")
for _ in range(2):
    x = P.plan(0).siddon_back(y)
torch.cuda.synchronize()
