for cfg in "0 oi" "1 o" "1 oi" "2 o" "2 oi"; do set -- $cfg
echo "pf=$1 set=$2 eval: $(ALORA_ATTN_PF=$1 ALORA_ATTN_PF_SET=$2 timeout 300 python scratch/fwd_step.py 12 20 2032 1 2>&1 | tail -1)"
echo "pf=$1 set=$2 dec : $(ALORA_ATTN_PF=$1 ALORA_ATTN_PF_SET=$2 timeout 300 python scratch/fwd_step.py 12 1 2048 1 2>&1 | tail -1)"
done
