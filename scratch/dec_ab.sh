timeout 600 python -m pytest tests -q -m gpu -x 2>&1 | tail -3
for i in 1 2; do
echo "new: $(timeout 300 python scratch/fwd_step.py 12 1 2048 1 2>&1 | tail -1)"
echo "old: $(ALORA_ATTN_NO_DECODE=1 timeout 300 python scratch/fwd_step.py 12 1 2048 1 2>&1 | tail -1)"
done
echo "skip-attn: $(ALORA_SKIP=attention timeout 300 python scratch/fwd_step.py 12 1 2048 1 2>&1 | tail -1)"
