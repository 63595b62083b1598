#!/bin/bash
# Per-tile timeline of the shared-prefix attention (ALORA_ATTN_TL=1, CTA (0,0), SM cycles) for the in-tree build
# and every variants/*.so, at the C3 eval step (2 layers).
for v in default $(cd paper_2512_17910_b200/variants 2>/dev/null && ls *.so | sed 's/\.so$//'); do
  if [ $v = default ]; then L=""; else L=paper_2512_17910_b200/variants/$v.so; fi
  echo "== $v"; ALORA_LIB=$L ALORA_ATTN_TL=1 GRAPH=0 timeout 300 python tools/eval_step.py c3 eval 1 2 2>&1 | grep -E "timeline" | tail -2
done
