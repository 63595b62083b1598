#!/bin/bash
for env in "ALORA_WS_BN=64 ALORA_WS_S=2" "ALORA_WS_BN=64 ALORA_WS_S=4" "ALORA_WS_BN=128 ALORA_WS_S=3" "X=1"; do
 for m in 240 129 256 12; do
  for nk in "2048 2048" "3072 2048" "2048 8192"; do
  echo "$env M=$m: $(env $env timeout 60 python scratch/ws_debug2.py $m $nk 20 2>&1 | grep -E 'bad|Error' | tail -1)"
  done
 done
done
timeout 600 python -m pytest tests -m gpu -x -q 2>&1 | tail -3
python scratch/fwd_step.py 12 20 2032 5 2>&1 | tail -1
python scratch/fwd_step.py 12 1 2048 5 2>&1 | tail -1
ALORA_PDL=0 python scratch/fwd_step.py 12 20 2032 5 2>&1 | tail -1
ALORA_GEMM_TRACE=1 ALORA_PDL=0 python scratch/fwd_step.py 12 20 2032 1 2>&1 | grep trace | tail -7 | cut -c1-250
