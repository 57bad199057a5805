#!/usr/bin/env bash
# ncu --set full of the three big kernels at configs[1] (one launch each, the
# second query: a speculative one), plus the launch list.
cd "${GRAFT_REPO_ROOT:-$(pwd)}"; mkdir -p gpurun_out
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:"k_trace_query|k_bounds|k_cross_stats" -s 3 -c 3 -f -o gpurun_out/prof_c1 python bench.py --steps 1 --warmup 1 --no-e2e --no-cpu-baseline > gpurun_out/ncu_c1.log 2>&1; echo "ncu rc=$?"
tail -2 gpurun_out/ncu_c1.log
