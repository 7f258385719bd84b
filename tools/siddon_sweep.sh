#!/bin/bash
# usage (GPU box): tools/siddon_sweep.sh variant...  -> C4 Siddon back time per variant
for v in "$@"; do
  if [ "$v" = default ]; then L=""; else L=build/variants/libctproj_b200_$v.so; fi
  CTPROJ_LIB=$L timeout 600 python - "$v" <<'PY'
import json, sys, torch
sys.path.insert(0, ".")
import paper_2307_05801_b200 as ct
from paper_2307_05801_b200 import configs
g, spec = ct.parse_config(json.dumps(configs.c4()))
plan = ct.ProjectorPair(ct.SIDDON, g, spec).plan(0)
y = torch.rand((1,) + g.shape, device="cuda")
x = torch.rand((1,) + spec.shape, device="cuda")
plan.siddon_back(y); plan.siddon_forward(x); torch.cuda.synchronize()
e0, e1, e2 = (torch.cuda.Event(enable_timing=True) for _ in range(3))
e0.record(); plan.siddon_back(y); e1.record(); plan.siddon_forward(x); e2.record(); torch.cuda.synchronize()
print(sys.argv[1], "c4_back_ms", round(e0.elapsed_time(e1), 1), "c4_fwd_ms", round(e1.elapsed_time(e2), 1))
PY
done
