timeout 900 python -m pytest tests -q -m gpu -x 2>&1 | tail -1
for i in 1 2; do
echo "cc eval:  $(FORCE_GRAPH=1 timeout 300 python scratch/fwd_step.py 12 20 2032 3 2>&1 | tail -1)"
echo "gemm eval: $(ALORA_SHRINK_GEMM=1 FORCE_GRAPH=1 timeout 300 python scratch/fwd_step.py 12 20 2032 3 2>&1 | tail -1)"
echo "cc dec:   $(timeout 300 python scratch/fwd_step.py 12 1 2048 3 2>&1 | tail -1)"
echo "gemm dec: $(ALORA_SHRINK_GEMM=1 timeout 300 python scratch/fwd_step.py 12 1 2048 3 2>&1 | tail -1)"
done
