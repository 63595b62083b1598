timeout 600 python -m pytest tests/test_gpu_bf16_model.py tests/test_gpu_graphs.py -q -x 2>&1 | tail -1
for i in 1 2; do
echo "whole: $(timeout 300 python scratch/fwd_step.py 12 1 2048 1 2>&1 | tail -1)"
echo "split: $(ALORA_DEC_WHOLE_MIN=100000 timeout 300 python scratch/fwd_step.py 12 1 2048 1 2>&1 | tail -1)"
done
