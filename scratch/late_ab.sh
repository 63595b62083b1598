timeout 600 python -m pytest tests -q -m gpu -x 2>&1 | tail -3
for i in 1 2; do
echo "late: $(timeout 300 python scratch/fwd_step.py 12 20 2032 1 2>&1 | tail -1)"
echo "nolate: $(ALORA_NO_LATE_WAIT=1 timeout 300 python scratch/fwd_step.py 12 20 2032 1 2>&1 | tail -1)"
done
echo "dec: $(timeout 300 python scratch/fwd_step.py 12 1 2048 1 2>&1 | tail -1)"
