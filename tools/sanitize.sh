#!/usr/bin/env bash
# compute-sanitizer memcheck, racecheck, initcheck and synccheck over the GPU parity tests (small shapes).
cd "$(dirname "$0")/.."
mkdir -p gpurun_out/sanitize
CS=/usr/local/cuda/bin/compute-sanitizer
for tool in ${TOOLS:-memcheck racecheck initcheck synccheck}; do
  timeout 1500 $CS --tool $tool --print-limit 20 --error-exitcode 9 \
    python -m pytest tests/test_gpu_parity.py tests/test_gpu_api.py tests/test_coselect.py -m gpu -x -q -p no:cacheprovider \
    > gpurun_out/sanitize/$tool.log 2>&1
  echo "$tool rc=$?" >> gpurun_out/sanitize/summary.txt
done
cat gpurun_out/sanitize/summary.txt
