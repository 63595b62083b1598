timeout 600 python -m pytest tests -q -m gpu -x 2>&1 | tail -5
for i in 1; do ALORA_ATTN_TRACE=1 timeout 300 python scratch/fwd_step.py 12 20 2032 1 2>&1 | grep "attn trace" | tail -2; done
timeout 300 python scratch/fwd_step.py 12 20 2032 1 2>&1 | tail -1
