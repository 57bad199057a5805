#!/usr/bin/env bash
# A/B of the whole device-resident query step (bench.py, no e2e / CPU legs):
# the in-tree build and every build/variants/*.so, REPS rounds interleaved.
cd "${GRAFT_REPO_ROOT:-$(pwd)}"
mkdir -p gpurun_out
: > gpurun_out/ab_bench.txt
for rep in $(seq ${REPS:-2}); do
  for v in base build/variants/*.so; do
    if [ "$v" = base ]; then unset PSG_LIB; n=base; else export PSG_LIB=$v; n=$(basename $v .so); fi
    l=$(timeout 600 python bench.py --steps ${STEPS:-10} --warmup 3 --no-e2e --no-cpu-baseline 2>/dev/null | grep '^{')
    echo "$n $(python -c "import json,sys; d=json.loads(sys.argv[1]); print(round(d['ms_per_step'],3), round(d['roofline']['kernel_ms'],3), round(d['roofline']['pass1_k_bounds_ms'],3))" "$l")" >> gpurun_out/ab_bench.txt
  done
done
cat gpurun_out/ab_bench.txt
