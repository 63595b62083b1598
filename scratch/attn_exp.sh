for e in 0 3 4 5; do echo "exp=$e"; ALORA_ATTN_EXP=$e ALORA_ATTN_TRACE=1 python scratch/fwd_step.py 12 20 2032 1 2>&1 | grep "attn trace" | tail -1; done
