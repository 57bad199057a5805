#!/usr/bin/env bash
# Evidence pass: GPU parity suite, the default bench line (device + e2e + CPU
# baseline), the reference arm, the ncu launch list of the bench command, and
# ncu --set full captures of the three main kernels (10k traces).
cd "${GRAFT_REPO_ROOT:-$(pwd)}"
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?"; tail -2 gpurun_out/pytest_gpu.log
timeout 1200 python bench.py > gpurun_out/bench_full.log 2>&1; echo "bench rc=$?"; grep '^{' gpurun_out/bench_full.log | tail -1 | cut -c1-300
timeout 900 python bench.py --impl reference > gpurun_out/bench_ref.log 2>&1; echo "ref rc=$?"; grep '^{' gpurun_out/bench_ref.log | tail -1 | cut -c1-300
STAGES=ncu_list bash tools/gpu_round.sh > /dev/null 2>&1; echo "ncu_list done"
KREGEX="k_trace_query|k_bounds|k_cross_stats" SKIP=3 COUNT=3 OUT=prof_all bash tools/ncu_query.sh
