#!/bin/bash
# launch list + full ncu captures of the aLoRA C2 eval forward (scratch/fwd_step.py)
mkdir -p gpurun_out
python scratch/fwd_step.py 12 20 2032 5 > gpurun_out/fwd_plain.log 2>&1
# warm-up = 3 forwards; each forward ~ 180 launches
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -s 700 -c 180 --csv --log-file gpurun_out/fwd_launches.csv python scratch/fwd_step.py 12 20 2032 1 > /dev/null 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:attn_tc -s 40 -c 2 -o gpurun_out/prof_attn -f python scratch/fwd_step.py 12 20 2032 1 > gpurun_out/ncu_attn.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:gemm_bf16 -s 200 -c 6 -o gpurun_out/prof_gemm -f python scratch/fwd_step.py 12 20 2032 1 > gpurun_out/ncu_gemm.log 2>&1
timeout 900 ncu --set full --clock-control none -k regex:"rmsnorm|kv_write|embed|argmax" -s 40 -c 8 -o gpurun_out/prof_small -f python scratch/fwd_step.py 12 20 2032 1 > gpurun_out/ncu_small.log 2>&1
ls -la gpurun_out
