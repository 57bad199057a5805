cd "${GRAFT_REPO_ROOT:-$(pwd)}"; mkdir -p gpurun_out
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_trace_query -s 1 -c 1 -f -o gpurun_out/prof_il python bench.py --traces 10000 --steps 1 --warmup 1 --no-e2e --no-cpu-baseline > gpurun_out/ncu_il.log 2>&1; echo "ncu rc=$?"
PSG_LIB=build/variants/r8.so timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_trace_query -s 1 -c 1 -f -o gpurun_out/prof_r8 python bench.py --traces 10000 --steps 1 --warmup 1 --no-e2e --no-cpu-baseline > gpurun_out/ncu_r8.log 2>&1; echo "ncu rc=$?"
REPS=1 STEPS=10 bash tools/ab_bench.sh
