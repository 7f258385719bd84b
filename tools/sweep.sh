#!/bin/bash
# usage (on the GPU box): tools/sweep.sh variant1 variant2 ...   ("default" = in-tree library)
# prints one line per variant: GUPS and per-kernel ms (C3, 2 timed steps)
for v in "$@"; do
  if [ "$v" = default ]; then L=""; else L=build/variants/libctproj_b200_$v.so; fi
  out=$(CTPROJ_LIB=$L timeout 300 python bench.py --steps 2 --warmup 1 --no-cpu --no-e2e ${SWEEP_ARGS} 2>&1 | tail -1)
  echo "$out" | python -c "
import json,sys
try:
    d=json.loads(sys.stdin.read()); k=d['kernels']
    print('$v', round(d['value'],2), 'fwd_ms', k['sf_forward_kernel']['ms'], 'back_ms', k['sf_back_kernel']['ms'])
except Exception as e:
    print('$v FAILED', e)
" || echo "$v: $out"
done
