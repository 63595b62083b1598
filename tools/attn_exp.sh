#!/bin/bash
# Attention bottleneck experiments at the C3 eval step (4 layers): per-kernel profile with the tensor-core MMAs
# switched off (ALORA_ATTN_EXP=64; outputs are wrong, only times are read), the per-CTA phase trace, and the
# one-query-tile variant.
set -u
L=${L:-4}
for e in 0 64; do
  echo "== ALORA_ATTN_EXP=$e"
  ALORA_ATTN_EXP=$e PROFILE=1 timeout 300 python tools/eval_step.py c3 eval 5 $L 2>&1 | grep -E "step|attention"
done
echo "== MT=1"
ALORA_ATTN_MT=1 PROFILE=1 timeout 300 python tools/eval_step.py c3 eval 5 $L 2>&1 | grep -E "step|attention"
echo "== trace"
ALORA_ATTN_TRACE=1 timeout 300 python tools/eval_step.py c3 eval 1 2 2>&1 | grep -E "trace" | tail -2
