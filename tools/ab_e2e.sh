#!/usr/bin/env bash
# A/B of bench.py e2e flags in one box: ARGSETS="-;--prefetch" (';'-separated,
# "-" = none), REPS rounds interleaved; prints e2e s/step and the H2D rate.
cd "${GRAFT_REPO_ROOT:-$(pwd)}"; mkdir -p gpurun_out
: > gpurun_out/ab_e2e.txt
IFS=';' read -ra SETS <<< "${ARGSETS:--}"
for rep in $(seq ${REPS:-3}); do
  for set in "${SETS[@]}"; do
    l=$(timeout 900 python bench.py --steps 3 --warmup 3 --no-cpu-baseline $( [ "$set" = "-" ] || echo $set ) 2>/dev/null | grep '^{')
    echo "[$set] $(python -c "import json,sys; d=json.loads(sys.argv[1])['e2e']; print(round(d['s_per_step'],4), round(d['roofline']['h2d_gbs'],2), round(d['roofline']['frac'],3))" "$l")" >> gpurun_out/ab_e2e.txt
  done
done
cat gpurun_out/ab_e2e.txt
