#!/bin/bash
for m in 240 129 256 12; do
  for nk in "2048 2048" "3072 2048" "2048 8192" "384 2048"; do
  echo "M=$m: $(timeout 60 python scratch/ws_debug2.py $m $nk 10 2>&1 | grep -E 'bad|Error' | tail -1)"
  done
done
timeout 600 python -m pytest tests -m gpu -x -q 2>&1 | tail -3
python scratch/fwd_step.py 12 20 2032 5 2>&1 | tail -1
python scratch/fwd_step.py 12 1 2048 5 2>&1 | tail -1
ALORA_GEMM_TRACE=1 ALORA_PDL=0 python scratch/fwd_step.py 12 20 2032 1 2>&1 | grep trace | tail -7 | cut -c1-250
ALORA_GEMM_TRACE=1 ALORA_PDL=0 python scratch/fwd_step.py 12 1 2048 1 2>&1 | grep trace | tail -7 | cut -c1-250
