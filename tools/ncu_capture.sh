cd ${GRAFT_REPO_ROOT}
mkdir -p gpurun_out
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_trace_query|k_bounds|k_cross_stats" -s 3 -c 3 -f -o gpurun_out/prof_all python bench.py --traces 10000 --steps 1 --warmup 1 --no-e2e --no-cpu-baseline > gpurun_out/ncu_full.log 2>&1; echo rc=$?
tail -3 gpurun_out/ncu_full.log
