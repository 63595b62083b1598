for i in $(seq 1 6); do timeout 120 python -m pytest tests/test_gpu_bf16_model.py -k paged -q -x 2>&1 | tail -1; done; bash scratch/attn_ab2.sh
