#!/bin/bash
mkdir -p gpurun_out
ALORA_ATTN_TRACE=1 ALORA_GEMM_TRACE=1 python scratch/fwd_step.py 12 20 2032 1 > gpurun_out/trace.log 2>&1
python scratch/gemm_micro.py > gpurun_out/gemm_micro.log 2>&1
tail -3 gpurun_out/trace.log
