#!/usr/bin/env bash
# configs[4] (C5) sweep on one GPU: 10k / 100k / 1M traces x 10,050 events
# (150 iterations x 67), device-resident query; one JSON line per size.
cd "${GRAFT_REPO_ROOT:-$(pwd)}"
mkdir -p gpurun_out
for n in 10000 100000 1000000; do
  timeout 900 python bench.py --traces $n --iters 150 --steps 3 --warmup 3 --no-e2e --no-cpu-baseline \
    > gpurun_out/c5_$n.log 2>&1
  echo "n=$n rc=$?"; grep '^{' gpurun_out/c5_$n.log | tail -1 | cut -c1-400; tail -2 gpurun_out/c5_$n.log | grep -v '^{' | cut -c1-300
done
