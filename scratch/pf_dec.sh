timeout 900 python -m pytest tests -q -m gpu -x 2>&1 | tail -1
for i in 1 2 3; do
echo "pf:   $(timeout 300 python scratch/fwd_step.py 12 1 2048 3 2>&1 | tail -1)"
echo "nopf: $(ALORA_NO_L2_PREFETCH=1 timeout 300 python scratch/fwd_step.py 12 1 2048 3 2>&1 | tail -1)"
done
