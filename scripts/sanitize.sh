#!/bin/bash
# compute-sanitizer over the kernel and reader GPU tests (B200). Logs under
# gpurun_out/sanitize_*.log; run from the repo root.
set -u
mkdir -p gpurun_out
CS=/usr/local/cuda/bin/compute-sanitizer
for tool in memcheck synccheck racecheck initcheck; do
  timeout 1500 $CS --tool $tool --target-processes all --print-limit 50 --error-exitcode 99 \
    python -m pytest tests/test_gpu_kernels.py tests/test_gpu_reader.py tests/test_gpu_teacher_reply.py \
    -m gpu -q -x -p no:cacheprovider > gpurun_out/sanitize_$tool.log 2>&1
  echo "$tool exit=$?" >> gpurun_out/sanitize_summary.txt
done
