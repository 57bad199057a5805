#!/usr/bin/env bash
# TEST INFRASTRUCTURE: links tests/dropin/dropin_test.cpp with the drop-in
# binding (integration/_build/libperfslice_gpu.a), libpsg.so and the
# reference core built by oracle/build_ref.sh (the checker).  Output:
# tests/dropin/_build/dropin_test (git-ignored, travels to the GPU box).
set -euo pipefail
HERE="$(cd "$(dirname "$0")" && pwd)"
ROOT="$(cd "$HERE/../.." && pwd)"
R=${PERFSLICE_REF:-/root/reference/proj}
O="$HERE/_build"
if [ ! -d "$R/src/core" ]; then
  echo "tests/dropin/build.sh: $R not present; keeping prebuilt $O" >&2
  exit 0
fi
mkdir -p "$O"
g++ -std=c++20 -O2 -I"$R/src" -I"$R/src/core" -I"$R/tests" -I"$ROOT/oracle/_ref/shim" \
    -I"$ROOT/include" -I"$ROOT/integration" "$HERE/dropin_test.cpp" \
    "$ROOT/integration/_build/libperfslice_gpu.a" "$ROOT/oracle/_ref/libperfslice_core.a" \
    -L"$ROOT/paper_2605_03561_b200" -lpsg -Wl,-rpath,'$ORIGIN/../../../paper_2605_03561_b200' \
    -lpthread -o "$O/dropin_test"
echo "tests/dropin/build.sh: ok -> $O/dropin_test"
