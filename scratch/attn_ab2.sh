timeout 600 python -m pytest tests -q -m gpu -x 2>&1 | tail -2
ALORA_ATTN_TRACE=1 timeout 300 python scratch/fwd_step.py 12 20 2032 1 2>&1 | grep "attn trace" | tail -2
for i in 1 2; do
echo "new: $(timeout 300 python scratch/fwd_step.py 12 20 2032 1 2>&1 | tail -1)"
echo "old: $(ALORA_LIB=scratch/libs/old_attn.so timeout 300 python scratch/fwd_step.py 12 20 2032 1 2>&1 | tail -1)"
done
