#!/usr/bin/env bash
# A/B of pass 1 (k_bounds) settings: ENVS as in ab_env.sh; prints step ms,
# k_trace_query ms and k_bounds ms per run.
cd "${GRAFT_REPO_ROOT:-$(pwd)}"; mkdir -p gpurun_out
: > gpurun_out/ab_bounds.txt
IFS=';' read -ra SETS <<< "${ENVS:--}"
for rep in $(seq ${REPS:-2}); do
  for set in "${SETS[@]}"; do
    l=$(env $( [ "$set" = "-" ] || echo $set ) timeout 600 python bench.py --steps ${STEPS:-10} --warmup 3 --no-e2e --no-cpu-baseline 2>/dev/null | grep '^{')
    echo "[$set] $(python -c "import json,sys; d=json.loads(sys.argv[1]); r=d['roofline']; print(round(d['ms_per_step'],3), round(r['kernel_ms'],3), round(r['pass1_k_bounds_ms'],3), d['clocks']['sm_mhz'])" "$l")" >> gpurun_out/ab_bounds.txt
  done
done
cat gpurun_out/ab_bounds.txt
