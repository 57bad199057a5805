#!/usr/bin/env bash
# A/B: the breakdown for the in-tree build and every build/variants/*.so
cd "${GRAFT_REPO_ROOT:-$(pwd)}"
mkdir -p gpurun_out
N=${1:-10000}
echo "base $(python tools/breakdown.py $N)" > gpurun_out/ab.txt
for v in build/variants/*.so; do
  echo "$(basename $v .so) $(PSG_LIB=$v python tools/breakdown.py $N)" >> gpurun_out/ab.txt
done
cat gpurun_out/ab.txt
