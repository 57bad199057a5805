#!/usr/bin/env bash
# ncu --set full of one k_trace_query launch at the C5 shape (150 iterations
# per trace), base build and build/variants/r8.so
cd "${GRAFT_REPO_ROOT:-$(pwd)}"; mkdir -p gpurun_out
N=${NTR:-20000}
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_trace_query -s 1 -c 1 -f \
  -o gpurun_out/prof_c5_il python bench.py --traces $N --iters 150 --steps 1 --warmup 1 --no-e2e --no-cpu-baseline > /dev/null 2>&1; echo rc=$?
PSG_LIB=build/variants/r8.so timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_trace_query -s 1 -c 1 -f \
  -o gpurun_out/prof_c5_r8 python bench.py --traces $N --iters 150 --steps 1 --warmup 1 --no-e2e --no-cpu-baseline > /dev/null 2>&1; echo rc=$?
