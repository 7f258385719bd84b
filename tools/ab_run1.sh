#!/bin/bash
# usage (on the GPU box): DIRS=f CFG=c3 tools/ab_run1.sh base new v2 ...
#   kernel times + output digests of each library variant ("new" = the
#   in-tree library, else build/variants/libctproj_b200_<name>.so), then
#   every variant's outputs compared against the first one's.
O=gpurun_out/ab1; mkdir -p $O
DIRS=${DIRS:-fb}; CFG=${CFG:-c3}
for v in "$@"; do
  if [ $v = new ]; then L=""; else L=build/variants/libctproj_b200_$v.so; fi
  CTPROJ_LIB=$L timeout 300 python tools/ab_probe.py --config $CFG --dirs $DIRS --tag $v --out $O 2>&1 | tail -1
done
for v in "${@:2}"; do echo "$v vs $1: $(python tools/ab_probe.py --compare $O/$v.npz $O/$1.npz)"; done
