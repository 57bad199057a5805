#!/usr/bin/env bash
# One ncu --set full capture of k_trace_query (10k traces, second launch).
cd "${GRAFT_REPO_ROOT:-$(pwd)}"
mkdir -p gpurun_out
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"${KREGEX:-k_trace_query}" -s ${SKIP:-1} -c ${COUNT:-1} -f \
  -o gpurun_out/${OUT:-prof_q} python bench.py --traces 10000 --steps 1 --warmup 1 --no-e2e --no-cpu-baseline \
  > gpurun_out/ncu_q.log 2>&1; echo "ncu rc=$?"
