#!/usr/bin/env bash
# Builds the reference's public C ABI (proj/src/capi.cpp -> libperfslice.so)
# with the GPU underneath: the reference's own sources, with the two call
# sites INTEGRATION.md §2 switches, compiled next to the drop-in binding and
# linked against libpsg.so.  Output: integration/_build/public_abi/libperfslice.so
# (git-ignored; travels to the GPU box).  The sources are read where they lie;
# only the two patched translation units are written (sed) into _build.
#
#   query.cpp:338      ingest::read_slices(...)          -> perfslice::gpu::read_slices(...)
#   workflows.cpp:215  itermodel::build_tri_model(...)   -> perfslice::gpu::build_tri_model(...)
#   workflows.cpp:303  (imbalance_report, iterations_report)
#
# Everything else (session cache, diagnostics, clustering, report rendering,
# the ps_* entry points and their error mapping) is the reference's code.
set -euo pipefail
HERE="$(cd "$(dirname "$0")" && pwd)"
ROOT="$(dirname "$HERE")"
R=${PERFSLICE_REF:-/root/reference/proj}
O="$HERE/_build/public_abi"
if [ ! -d "$R/src/core" ]; then
  echo "integration/build_public_abi.sh: $R not present; keeping prebuilt $O" >&2
  exit 0
fi
SHIM="$ROOT/oracle/_ref/shim"   # nlohmann single header (oracle/build_ref.sh)
[ -f "$SHIM/nlohmann/json.hpp" ] || "$ROOT/oracle/build_ref.sh" > /dev/null
mkdir -p "$O/patched" "$O/obj"
sed -e 's/ingest::read_slices(\*db_, requests, jobs_)/perfslice::gpu::read_slices(*db_, requests, jobs_)/' \
    -e 's/#include "query.hpp"/#include "query.hpp"\n#include "perfslice_gpu.hpp"/' \
    "$R/src/core/query.cpp" > "$O/patched/query.cpp"
sed -e 's/itermodel::build_tri_model(/perfslice::gpu::build_tri_model(/g' \
    -e 's/#include "workflows.hpp"/#include "workflows.hpp"\n#include "perfslice_gpu.hpp"/' \
    "$R/src/core/workflows.cpp" > "$O/patched/workflows.cpp"
grep -q "perfslice::gpu::read_slices" "$O/patched/query.cpp"
[ "$(grep -c "perfslice::gpu::build_tri_model" "$O/patched/workflows.cpp")" = 2 ]
cp "$R/src/core/synthgen.cpp" "$O/patched/synthgen.cpp.orig"
sed -e '415s/{{}})/std::vector<double>{})/' -e '432s/{{}})/std::vector<uint32_t>{})/' \
    -e '443s/{{}})/std::vector<std::string>{})/' "$R/src/core/synthgen.cpp" > "$O/patched/synthgen.cpp"
rm -f "$O/patched/synthgen.cpp.orig"
CXX="g++ -std=c++20 -O2 -fPIC -w -I$R/src/core -I$R/src -I$SHIM -I$ROOT/include -I$HERE"
pids=()
for f in common util store frame ingest itermodel diagnostics topology; do
  $CXX -c "$R/src/core/$f.cpp" -o "$O/obj/$f.o" & pids+=($!)
done
for f in query workflows synthgen; do
  $CXX -c "$O/patched/$f.cpp" -o "$O/obj/$f.o" & pids+=($!)
done
$CXX -c "$HERE/perfslice_gpu.cpp" -o "$O/obj/perfslice_gpu.o" & pids+=($!)
for p in "${pids[@]}"; do wait "$p"; done
g++ -std=c++20 -O2 -shared -fPIC -I$R/include -I$R/src -I$SHIM "$R/src/capi.cpp" "$O"/obj/*.o \
    -L"$ROOT/paper_2605_03561_b200" -lpsg -Wl,-rpath,'$ORIGIN/../../../paper_2605_03561_b200' \
    -lpthread -o "$O/libperfslice.so"
echo "integration/build_public_abi.sh: ok -> $O/libperfslice.so"
