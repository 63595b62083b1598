#!/bin/bash
# A/B the in-tree library against variants/*.so on the C3 eval step (4 layers): attention time per build.
# usage: tools/ab_libs.sh [c2|c3] [eval|decode] [layers] [lib names...]
set -u
cfg=${1:-c3}; mode=${2:-eval}; L=${3:-4}; shift 3 || true
libs=${*:-$(cd paper_2512_17910_b200/variants 2>/dev/null && ls *.so | sed 's/\.so$//')}
for rep in 1 2; do
  echo "== default"
  PROFILE=1 timeout 300 python tools/eval_step.py $cfg $mode 5 $L 2>&1 | grep -E "step|attention " | head -2
  for v in $libs; do
    echo "== $v"
    ALORA_LIB=paper_2512_17910_b200/variants/$v.so PROFILE=1 timeout 300 python tools/eval_step.py $cfg $mode 5 $L 2>&1 | grep -E "step|attention " | head -2
  done
done
