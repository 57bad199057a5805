cd "${GRAFT_REPO_ROOT:-$(pwd)}"; mkdir -p gpurun_out
for v in base build/variants/r8.so; do
  if [ "$v" = base ]; then unset PSG_LIB; else export PSG_LIB=$v; fi
  for n in 10000 100000; do
    l=$(timeout 600 python bench.py --traces $n --iters 150 --steps 5 --warmup 3 --no-e2e --no-cpu-baseline 2>/dev/null | grep '^{')
    echo "$(basename $v) n=$n $(python -c "import json,sys; d=json.loads(sys.argv[1]); print(round(d['ms_per_step'],3), round(d['roofline']['kernel_ms'],3), d['value'])" "$l")"
  done
done
unset PSG_LIB
timeout 600 python tools/sparse_bench.py 2000 50000 > gpurun_out/sparse_bench.json 2>&1; tail -1 gpurun_out/sparse_bench.json
