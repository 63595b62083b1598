#!/bin/bash
timeout 600 python -m pytest tests -m gpu -q -x 2>&1 | tail -3
python scratch/fwd_step.py 12 20 2032 5 2>&1 | tail -1
python scratch/fwd_step.py 12 1 2048 5 2>&1 | tail -1
ALORA_GEMM_TRACE=1 ALORA_PDL=0 python scratch/fwd_step.py 12 20 2032 1 2>&1 | grep trace | tail -6 | cut -c1-250
timeout 300 python bench.py --steps 3 --warmup 3 --no-cpu-baseline --lora-steps 1 2>&1 | tail -1 | python -c "
import json,sys; d=json.loads(sys.stdin.read()); print('value',d['value'],'ms',d['ms_per_step'],'e2e',d['e2e']['value']); print('alora',d['alora']); print('lora',d['lora']); print({k:(v['us_per_launch'],v['launches']) for k,v in d['kernels'].items()})"
