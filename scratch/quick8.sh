#!/bin/bash
timeout 600 python -m pytest tests -m gpu -q -x 2>&1 | tail -3
timeout 120 python __graft_entry__.py smoke 2>&1 | tail -2
python scratch/fwd_step.py 12 20 2032 5 2>&1 | tail -1
python scratch/fwd_step.py 12 1 2048 5 2>&1 | tail -1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -s 700 -c 200 --csv --log-file gpurun_out/dec_launches.csv python scratch/fwd_step.py 12 1 2048 1 > /dev/null 2>&1
python scratch/launches.py gpurun_out/dec_launches.csv
