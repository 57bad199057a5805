cd "${GRAFT_REPO_ROOT:-$(pwd)}"
for v in base build/variants/wcta.so; do
  if [ "$v" = base ]; then unset PSG_LIB; n=base; else export PSG_LIB=$v; n=$(basename $v .so); fi
  timeout 600 ncu --metrics gpu__time_duration.sum,smsp__inst_executed.sum,sm__warps_active.avg.pct_of_peak_sustained_active,launch__occupancy_limit_shared_mem,launch__occupancy_limit_registers,launch__occupancy_limit_blocks,launch__shared_mem_per_block_dynamic,smsp__issue_active.avg.pct_of_peak_sustained_active,launch__registers_per_thread --clock-control none -k regex:k_trace_query -s 2 -c 1 --csv python tools/breakdown.py ${NTR:-10000} ${FLAV:-full} 2>/dev/null | grep -v "^==" > gpurun_out/ncuab_$n.csv
done
