for k in none attention gemm_mlp_in gemm_mlp_out gemm_o gemm_qkv qkv_finalize rmsnorm lora_shrink gemm_lm_head attention,gemm_mlp_in,gemm_mlp_out,gemm_o,gemm_qkv,qkv_finalize,rmsnorm,lora_shrink,gemm_lm_head; do
echo "skip=$k $(ALORA_SKIP=$k timeout 300 python tools/fwd_step.py 12 20 2032 1 2>&1 | tail -1)"
done
echo "decode:"
for k in none attention gemm_mlp_in gemm_mlp_out gemm_o gemm_qkv qkv_finalize rmsnorm lora_shrink gemm_lm_head; do
echo "skip=$k $(ALORA_SKIP=$k timeout 300 python tools/fwd_step.py 12 1 2048 1 2>&1 | tail -1)"
done
