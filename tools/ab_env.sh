#!/bin/bash
# A/B environment settings on the eval step: tools/ab_env.sh <c2|c3> <eval|decode> <layers> <grep-regex> "ENV=.." ...
# each setting runs twice (alternating); prints the forward time and the per-kernel lines matching the regex.
cfg=$1; mode=$2; L=$3; pat=$4; shift 4
for rep in 1 2; do
  for e in "$@"; do
    echo "== $e"
    env $e PROFILE=1 timeout 300 python tools/eval_step.py $cfg $mode 5 $L 2>&1 | grep -E "step|$pat"
  done
done
