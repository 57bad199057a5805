cd "${GRAFT_REPO_ROOT:-$(pwd)}"
for it in 150 746; do
for v in base build/variants/*.so; do
  if [ "$v" = base ]; then unset PSG_LIB; n=base; else export PSG_LIB=$v; n=$(basename $v .so); fi
  for sh in one wide; do
    l=$(PSG_CTA_SHAPE=$sh timeout 600 python bench.py --traces 100000 --iters $it --steps 10 --warmup 3 --no-e2e --no-cpu-baseline 2>/dev/null | grep '^{')
    echo "iters=$it $n $sh $(python -c "import json,sys; d=json.loads(sys.argv[1]); print(round(d['ms_per_step'],3), round(d['roofline']['kernel_ms'],3))" "$l")"
  done
done; done
