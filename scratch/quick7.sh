#!/bin/bash
timeout 600 python -m pytest tests -m gpu -q -x 2>&1 | tail -3
python scratch/fwd_step.py 12 20 2032 5 2>&1 | tail -1
python scratch/fwd_step.py 12 1 2048 5 2>&1 | tail -1
ALORA_ATTN_TRACE=1 python scratch/fwd_step.py 12 20 2032 1 2>&1 | grep "attn trace" | tail -2
ALORA_ATTN_TRACE=1 python scratch/fwd_step.py 12 1 2048 1 2>&1 | grep "attn trace" | tail -1
