#!/bin/bash
ALORA_GEMM_TRACE=1 ALORA_PDL=0 python scratch/fwd_step.py 12 1 2048 1 2>&1 | grep trace | tail -6 | cut -c1-250
ALORA_GEMM_TRACE=1 ALORA_PDL=0 python scratch/fwd_step.py 12 20 2032 1 2>&1 | grep trace | tail -6 | cut -c1-250
