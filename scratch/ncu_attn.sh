#!/bin/bash
mkdir -p gpurun_out
timeout 900 ncu --set full --import-source on --clock-control none --warp-sampling-interval 0 -k regex:attn_tc -s 40 -c 1 -o gpurun_out/prof_attn2 -f python scratch/fwd_step.py 12 20 2032 1 > gpurun_out/ncu_attn2.log 2>&1
tail -2 gpurun_out/ncu_attn2.log
