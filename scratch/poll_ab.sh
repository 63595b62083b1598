for p in 32 0 100 250 500; do
echo "poll=$p $(ALORA_ATTN_POLL=$p timeout 300 python scratch/fwd_step.py 12 20 2032 1 2>&1 | tail -1)"
echo "poll=$p $(ALORA_ATTN_POLL=$p ALORA_PDL=0 ALORA_ATTN_TRACE=1 timeout 300 python scratch/fwd_step.py 12 20 2032 1 2>&1 | grep 'attn trace' | tail -1)"
done
