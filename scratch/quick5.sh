#!/bin/bash
python scratch/fwd_step.py 12 20 2032 5 2>&1 | tail -1
python scratch/fwd_step.py 12 1 2048 5 2>&1 | tail -1
ALORA_PDL=0 python scratch/fwd_step.py 12 20 2032 5 2>&1 | tail -1
