for i in $(seq 1 8); do timeout 300 python -m pytest tests -q -m gpu -rf 2>&1 | grep -E "FAILED|passed|failed" | tail -3; done
