cd "${GRAFT_REPO_ROOT:-$(pwd)}"
for rep in 1 2; do
for v in base build/variants/*.so; do
  if [ "$v" = base ]; then unset PSG_LIB; n=base; else export PSG_LIB=$v; n=$(basename $v .so); fi
  l=$(timeout 600 python bench.py --traces 100000 --iters 150 --steps 10 --warmup 3 --no-e2e --no-cpu-baseline 2>/dev/null | grep '^{')
  echo "$n $(python -c "import json,sys; d=json.loads(sys.argv[1]); print(round(d['ms_per_step'],3), round(d['roofline']['kernel_ms'],3), round(d['roofline']['pass1_k_bounds_ms'],3))" "$l")"
done; done
