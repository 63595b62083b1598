#!/bin/bash
mkdir -p gpurun_out
python scratch/fwd_step.py 12 20 2032 5 > gpurun_out/fwd_plain.log 2>&1
ALORA_ATTN_TRACE=1 python scratch/fwd_step.py 12 20 2032 1 2>&1 | grep "attn trace" | tail -2 >> gpurun_out/fwd_plain.log
ALORA_ATTN_TRACE=1 python scratch/fwd_step.py 12 1 2048 1 2>&1 | grep "attn trace" | tail -1 >> gpurun_out/fwd_plain.log
python scratch/fwd_step.py 12 1 2048 5 >> gpurun_out/fwd_plain.log 2>&1
timeout 300 python -m pytest tests -m gpu -x -q -k "attention or forward" > gpurun_out/pt.log 2>&1; tail -2 gpurun_out/pt.log >> gpurun_out/fwd_plain.log
python scratch/gemm_micro.py >> gpurun_out/fwd_plain.log 2>&1
cat gpurun_out/fwd_plain.log
