timeout 600 python -m pytest tests -q -m gpu -x 2>&1 | tail -1
for i in 1 2; do
echo "new eval: $(timeout 300 python scratch/fwd_step.py 12 20 2032 1 2>&1 | tail -1)"
echo "old eval: $(ALORA_LIB=scratch/libs/old_attn.so timeout 300 python scratch/fwd_step.py 12 20 2032 1 2>&1 | tail -1)"
echo "new dec : $(timeout 300 python scratch/fwd_step.py 12 1 2048 1 2>&1 | tail -1)"
echo "old dec : $(ALORA_LIB=scratch/libs/old_attn.so timeout 300 python scratch/fwd_step.py 12 1 2048 1 2>&1 | tail -1)"
done
