#!/usr/bin/env bash
# A/B of the device-resident query step (bench.py, no e2e / CPU legs) under
# environment variants: VARIANTS="name:VAR=val,VAR2=val ..." (base = none),
# REPS rounds interleaved.  One line per run: ms/step, k_trace_query ms, pass-1 ms.
cd "${GRAFT_REPO_ROOT:-$(pwd)}"
mkdir -p gpurun_out
OUT=gpurun_out/ab_env.txt
: > $OUT
for rep in $(seq ${REPS:-2}); do
  for v in base ${VARIANTS}; do
    n=${v%%:*}; envs=""
    [ "$v" != base ] && envs=$(echo ${v#*:} | tr ',' ' ')
    l=$(env $envs timeout 600 python bench.py --steps ${STEPS:-10} --warmup 3 --no-e2e --no-cpu-baseline ${BENCH_ARGS} 2>/dev/null | grep '^{')
    echo "$n $(python -c "import json,sys; d=json.loads(sys.argv[1]); r=d['roofline']; print(round(d['ms_per_step'],3), round(r['kernel_ms'],3), round(r['pass1_k_bounds_ms'],3))" "$l" 2>&1 | tail -1)" >> $OUT
  done
done
cat $OUT
