#!/usr/bin/env bash
# CTA-shape A/B of k_trace_query (PSG_CTA_SHAPE=one|wide) over trace lengths:
# 150 / 300 / 500 / 746 iterations of 67 events, 100k traces, device-resident.
cd "${GRAFT_REPO_ROOT:-$(pwd)}"
for it in 150 300 500 746; do
  for sh in one wide auto; do
    if [ $sh = auto ]; then unset PSG_CTA_SHAPE; else export PSG_CTA_SHAPE=$sh; fi
    l=$(timeout 600 python bench.py --traces 100000 --iters $it --steps 10 --warmup 3 --no-e2e --no-cpu-baseline 2>/dev/null | grep '^{')
    echo "iters=$it $sh $(python -c "import json,sys; d=json.loads(sys.argv[1]); print(round(d['ms_per_step'],3), round(d['roofline']['kernel_ms'],3))" "$l")"
  done
done
