#!/bin/bash
# launch list (one forward after 3 warm-up forwards) + full captures of the attention and the biggest GEMM
mkdir -p gpurun_out
python scratch/fwd_step.py 12 20 2032 5 > gpurun_out/fwd_plain.log 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -s 700 -c 200 --csv --log-file gpurun_out/fwd_launches.csv python scratch/fwd_step.py 12 20 2032 1 > /dev/null 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -s 700 -c 200 --csv --log-file gpurun_out/dec_launches.csv python scratch/fwd_step.py 12 1 2048 1 > /dev/null 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:attn_tc -s 40 -c 1 -o gpurun_out/prof_attn -f python scratch/fwd_step.py 12 20 2032 1 > gpurun_out/ncu_attn.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:gemm_ws -s 100 -c 5 -o gpurun_out/prof_gemm -f python scratch/fwd_step.py 12 20 2032 1 > gpurun_out/ncu_gemm.log 2>&1
python scratch/launches.py gpurun_out/fwd_launches.csv
python scratch/launches.py gpurun_out/dec_launches.csv
