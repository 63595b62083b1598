#!/bin/bash
# KV-partition sweep of the shared-prefix attention at one C3 step (ALORA_ATTN_PARTS forces the split count the
# planner would otherwise pick from its cost model). usage: tools/parts_sweep.sh <decode|eval> [parts...]
set -u
mode=$1; shift
for p in "$@"; do
  echo "== parts=$p"
  ALORA_ATTN_PARTS=$p PROFILE=1 timeout 300 python tools/eval_step.py c3 $mode 5 4 2>&1 | grep -E "step|attn|combine|merge"
done
