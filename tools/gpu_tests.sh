#!/usr/bin/env bash
# GPU-box pass: the GPU suite (or a -k selection via PYTEST_K) + the drop-in binary.
cd "${GRAFT_REPO_ROOT:-$(pwd)}"
mkdir -p gpurun_out
K=${PYTEST_K:-}
if [ -n "$K" ]; then
  timeout ${PYTEST_TIMEOUT:-1500} python -m pytest tests -m gpu -x -q -k "$K" > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?"
else
  timeout ${PYTEST_TIMEOUT:-1500} python -m pytest tests -m gpu -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?"
fi
tail -30 gpurun_out/pytest_gpu.log
