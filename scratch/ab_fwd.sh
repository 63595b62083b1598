for i in 1 2; do
echo "old"; ALORA_LIB=scratch/libs/old_attn.so timeout 300 python scratch/fwd_step.py 12 20 2032 1 2>&1 | tail -1
echo "new"; timeout 300 python scratch/fwd_step.py 12 20 2032 1 2>&1 | tail -1
done
