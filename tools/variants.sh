#!/usr/bin/env bash
# Builds tuning variants of libpsg.so into build/variants/<name>.so for A/B
# runs (PSG_LIB=build/variants/<name>.so python tools/breakdown.py).
#   tools/variants.sh name "-DPSG_RM=4 -DPSG_WMAX=8 ..." [name2 "defs2" ...]
set -euo pipefail
cd "$(dirname "$0")/.."
mkdir -p build/variants
NVCC=/usr/local/cuda/bin/nvcc
ARCH="-gencode arch=compute_100a,code=sm_100a"
while [ $# -ge 2 ]; do
  name=$1; defs=$2; shift 2
  o=build/variants/$name; mkdir -p $o
  for f in paper_2605_03561_b200/csrc/*.cu; do
    $NVCC $ARCH -O3 -std=c++17 -Iinclude -Ipaper_2605_03561_b200/csrc -lineinfo -Xcompiler -fPIC \
      --expt-relaxed-constexpr -diag-suppress 186 $defs -c $f -o $o/$(basename $f).o &
  done
  g++ -O3 -std=c++17 -Iinclude -Ipaper_2605_03561_b200/csrc -fPIC -I/usr/local/cuda/include $defs \
    -c paper_2605_03561_b200/csrc/psg_store.cpp -o $o/psg_store.cpp.o &
  wait
  $NVCC $ARCH -shared -cudart static -o build/variants/$name.so $o/*.o -ldl -lpthread
  echo "built build/variants/$name.so ($defs)"
done
