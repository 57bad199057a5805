#!/usr/bin/env bash
# Quick GPU iteration: parity suite, per-flavour kernel times (10k traces),
# device-resident bench at configs[1] (no e2e / CPU baseline).
cd "${GRAFT_REPO_ROOT:-$(pwd)}"
mkdir -p gpurun_out
if [ "${SKIP_TESTS:-0}" != 1 ]; then
  timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?"
  tail -15 gpurun_out/pytest_gpu.log
fi
timeout 300 python tools/breakdown.py 10000 > gpurun_out/bd.txt 2>&1; cat gpurun_out/bd.txt
timeout 600 python bench.py --no-e2e --no-cpu-baseline > gpurun_out/bench_full.log 2>&1; tail -c 1500 gpurun_out/bench_full.log
