#!/usr/bin/env bash
# ncu --set full of one k_trace_query launch at configs[1] shape, 10k traces
# (OUT=name, PSG_LIB=variant), for tools/regions.py and raw-metric comparisons.
cd "${GRAFT_REPO_ROOT:-$(pwd)}"; mkdir -p gpurun_out
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_trace_query -s 1 -c 1 -f \
  -o gpurun_out/${OUT:-prof_one} python bench.py --traces ${NTR:-10000} --steps 1 --warmup 1 --no-e2e --no-cpu-baseline \
  > gpurun_out/ncu_one.log 2>&1; echo "ncu rc=$?"
