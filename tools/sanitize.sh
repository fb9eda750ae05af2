#!/usr/bin/env bash
# compute-sanitizer over the small GPU tests (run under gpurun).  Logs -> gpurun_out/sanitize_*.log
set -u
export PATH=/usr/local/cuda/bin:$PATH
mkdir -p gpurun_out
OPS='gemm_bf16 and 1000 or resid_add_norm and 1000 or swiglu and 700 or rope and 900 or attention or embed or dh64 or row_scaled'
timeout 900 compute-sanitizer --tool memcheck --error-exitcode 3 python -m pytest tests/test_ops_gpu.py -q -k "$OPS" \
  > gpurun_out/sanitize_memcheck_ops.log 2>&1; echo "memcheck ops rc=$?"
timeout 900 compute-sanitizer --tool memcheck --error-exitcode 3 python -m pytest tests/test_parity_gpu.py -q \
  -k "test_model_parity_small and TINY_GQA and spread or last_layer or single_item" \
  > gpurun_out/sanitize_memcheck_model.log 2>&1; echo "memcheck model rc=$?"
timeout 900 compute-sanitizer --tool racecheck --error-exitcode 3 python -m pytest tests/test_ops_gpu.py -q \
  -k "gemm_bf16 and 1000 or resid_add_norm and 1000 or swiglu and 700 or rope and 900 or attention and 4-2-128 or dh64" \
  > gpurun_out/sanitize_racecheck.log 2>&1; echo "racecheck rc=$?"
timeout 900 compute-sanitizer --tool synccheck --error-exitcode 3 python -m pytest tests/test_ops_gpu.py -q \
  -k "gemm_bf16 and 1000 or attention and 4-2-128" > gpurun_out/sanitize_synccheck.log 2>&1; echo "synccheck rc=$?"
tail -n 3 gpurun_out/sanitize_*.log
