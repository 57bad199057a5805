#!/usr/bin/env bash
# Builds the drop-in binding (integration/perfslice_gpu.cpp) against the
# reference's headers into integration/_build/libperfslice_gpu.a — the object
# a reference maintainer links into their build next to libpsg.so (see
# INTEGRATION.md).  Needs the reference sources (PERFSLICE_REF, default
# /root/reference/proj); without them the prebuilt archive is kept.
set -euo pipefail
HERE="$(cd "$(dirname "$0")" && pwd)"
ROOT="$(dirname "$HERE")"
R=${PERFSLICE_REF:-/root/reference/proj}
O="$HERE/_build"
if [ ! -d "$R/src/core" ]; then
  echo "integration/build.sh: $R not present; keeping prebuilt $O" >&2
  exit 0
fi
mkdir -p "$O"
g++ -std=c++20 -O2 -fPIC -Wall -Wextra -I"$R/src" -I"$R/src/core" -I"$ROOT/include" \
    -c "$HERE/perfslice_gpu.cpp" -o "$O/perfslice_gpu.o"
rm -f "$O/libperfslice_gpu.a"
ar rcs "$O/libperfslice_gpu.a" "$O/perfslice_gpu.o"
echo "integration/build.sh: ok -> $O/libperfslice_gpu.a"
