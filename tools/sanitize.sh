#!/bin/bash
# compute-sanitizer passes over the -m gpu kernel/model tests (run on the GPU box; summaries -> gpurun_out/san_*.txt)
set -u
CS=/usr/local/cuda/bin/compute-sanitizer
OUT=${OUT:-gpurun_out}
mkdir -p $OUT
SMALL="tests/test_gpu_bf16_kernels.py tests/test_gpu_shared_prefix.py tests/test_gpu_bf16_model.py tests/test_gpu_graphs.py tests/test_gpu_pipelined.py"
run() {  # tool, log, pytest args...
  local tool=$1 log=$2; shift 2
  timeout ${SAN_TIMEOUT:-1500} $CS --tool $tool --print-limit 20 --error-exitcode 99 \
      python -m pytest -q -x -p no:cacheprovider "$@" > $OUT/$log 2>&1
  echo "$tool rc=$? $(grep -E 'ERROR SUMMARY|passed|failed' $OUT/$log | tail -2 | tr '\n' ' ')" | tee -a $OUT/san_summary.txt
}
run memcheck san_memcheck.txt $SMALL -k "not repeated"
run synccheck san_synccheck.txt tests/test_gpu_bf16_kernels.py tests/test_gpu_shared_prefix.py tests/test_gpu_bf16_model.py -k "not repeated and not pipeline"
run racecheck san_racecheck.txt tests/test_gpu_bf16_kernels.py tests/test_gpu_shared_prefix.py tests/test_gpu_bf16_model.py -k "attention or gemm or qkv"
run initcheck san_initcheck.txt tests/test_gpu_bf16_kernels.py tests/test_gpu_shared_prefix.py -k "not repeated"
