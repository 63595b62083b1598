#!/bin/bash
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,driver_version --format=csv > gpurun_out/smi.txt 2>&1
timeout 900 python -m pytest tests -q -m gpu > gpurun_out/final_tests.log 2>&1
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/final_smoke.log 2>&1
timeout 900 python bench.py > gpurun_out/bench.log 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -s 700 -c 170 --csv --log-file gpurun_out/fwd_launches.csv python scratch/fwd_step.py 12 20 2032 1 > /dev/null 2>&1
ALORA_GRAPHS=0 timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -s 700 -c 170 --csv --log-file gpurun_out/dec_launches.csv python scratch/fwd_step.py 12 1 2048 1 > /dev/null 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:attn_tc -s 40 -c 1 -o gpurun_out/prof_attn -f python scratch/fwd_step.py 12 20 2032 1 > gpurun_out/ncu_attn.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"gemm_ws|gemm_dec" -s 60 -c 6 -o gpurun_out/prof_gemm -f python scratch/fwd_step.py 12 20 2032 1 > gpurun_out/ncu_gemm.log 2>&1
ALORA_GRAPHS=0 timeout 900 ncu --set full --clock-control none --import-source on -k regex:gemm_dec -s 60 -c 6 -o gpurun_out/prof_dec -f python scratch/fwd_step.py 12 1 2048 1 > gpurun_out/ncu_dec.log 2>&1
ALORA_GRAPHS=0 timeout 900 ncu --set full --clock-control none --import-source on -k regex:attn_decode -s 20 -c 1 -o gpurun_out/prof_dec_attn -f python scratch/fwd_step.py 12 1 2048 1 > /dev/null 2>&1
tail -1 gpurun_out/final_tests.log; tail -1 gpurun_out/final_smoke.log
