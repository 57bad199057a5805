#!/usr/bin/env bash
# A/B of kernel DRAM traffic and time under ncu: base build and build/variants/*.so
# (CSV per variant in gpurun_out/ab_<name>.csv; summarise with tools/ab_ncu_summary.py)
cd "${GRAFT_REPO_ROOT:-$(pwd)}"
mkdir -p gpurun_out
K=${KREGEX:-k_bounds}
FLAV=${FLAV:-cube}
for v in base build/variants/*.so; do
  if [ "$v" = base ]; then unset PSG_LIB; n=base; else export PSG_LIB=$v; n=$(basename $v .so); fi
  timeout 600 ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum --clock-control none \
    -k regex:"$K" -s ${SKIP:-2} -c ${COUNT:-2} --csv --log-file gpurun_out/ab_$n.csv python tools/breakdown.py ${NTR:-10000} $FLAV > /dev/null 2>&1
  echo "$n rc=$?"
done
