#!/usr/bin/env bash
# A/B of environment settings on the in-tree build: ENVS="A=1 B=2;C=3" (one
# setting per ';'-separated entry, "-" = none), REPS rounds interleaved.
cd "${GRAFT_REPO_ROOT:-$(pwd)}"; mkdir -p gpurun_out
: > gpurun_out/ab_env.txt
IFS=';' read -ra SETS <<< "${ENVS:--}"
for rep in $(seq ${REPS:-2}); do
  for set in "${SETS[@]}"; do
    l=$(env $( [ "$set" = "-" ] || echo $set ) timeout 600 python bench.py --steps ${STEPS:-10} --warmup 3 --no-e2e --no-cpu-baseline ${ARGS:-} 2>/dev/null | grep '^{')
    echo "[$set] $(python -c "import json,sys; d=json.loads(sys.argv[1]); print(round(d['ms_per_step'],3), round(d['roofline']['kernel_ms'],3))" "$l")" >> gpurun_out/ab_env.txt
  done
done
cat gpurun_out/ab_env.txt
