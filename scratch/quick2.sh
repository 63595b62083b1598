#!/bin/bash
mkdir -p gpurun_out
timeout 600 python -m pytest tests -m gpu -x -q > gpurun_out/pt.log 2>&1; tail -15 gpurun_out/pt.log
python scratch/fwd_step.py 12 20 2032 5 2>&1 | tail -2
python scratch/fwd_step.py 12 1 2048 5 2>&1 | tail -2
ALORA_PDL=0 python scratch/fwd_step.py 12 20 2032 5 2>&1 | tail -1
ALORA_GEMM_TRACE=1 ALORA_PDL=0 python scratch/fwd_step.py 12 20 2032 1 2>&1 | grep trace | tail -8 | cut -c1-250
python scratch/gemm_micro.py 2>&1 | tail -16
