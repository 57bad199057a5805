#!/usr/bin/env bash
# Builds the UNMODIFIED reference core (/root/reference/proj) plus our harness
# (oracle/ref_harness.cpp) into oracle/_ref/ (git-ignored, travels to the GPU
# box with gpurun).  Test infrastructure only: the product never links this.
#
# Two shims, both outputs-only under oracle/_ref/ (nothing is copied into the
# tracked tree):
#   * nlohmann/json 3.11.3 single header from the cudnn_frontend thirdparty dir
#     plus a json_fwd.hpp forwarding header (the reference's vendor/ is absent);
#   * synthgen.cpp:415,432,443 use `{{}}` as a std::optional<std::vector<T>>
#     default, which GCC 13 rejects; a sed-generated copy in oracle/_ref/patched
#     spells the same empty vector as `std::vector<T>{}` (behaviour-identical).
# Usage: oracle/build_ref.sh  (no-op when /root/reference is absent)
set -euo pipefail
HERE="$(cd "$(dirname "$0")" && pwd)"
R=${PERFSLICE_REF:-/root/reference/proj}
O="$HERE/_ref"
if [ ! -d "$R/src/core" ]; then
  echo "build_ref: $R not present; keeping prebuilt $O" >&2
  exit 0
fi
NL=/opt/prime-rl/.venv/lib/python3.12/site-packages/include/cudnn_frontend/thirdparty/nlohmann/json.hpp
mkdir -p "$O/shim/nlohmann" "$O/patched" "$O/obj"
cp "$NL" "$O/shim/nlohmann/json.hpp"
printf '#pragma once\n#include "json.hpp"\n' > "$O/shim/nlohmann/json_fwd.hpp"
sed -e '415s/{{}})/std::vector<double>{})/' -e '432s/{{}})/std::vector<uint32_t>{})/' \
    -e '443s/{{}})/std::vector<std::string>{})/' "$R/src/core/synthgen.cpp" > "$O/patched/synthgen.cpp"
CXX="g++ -std=c++20 -O2 -fPIC -I$R/src/core -I$R/src -I$O/shim"
pids=()
for f in common util store frame ingest query itermodel diagnostics topology workflows; do
  $CXX -c "$R/src/core/$f.cpp" -o "$O/obj/$f.o" & pids+=($!)
done
$CXX -c "$O/patched/synthgen.cpp" -o "$O/obj/synthgen.o" & pids+=($!)
for p in "${pids[@]}"; do wait "$p"; done
rm -f "$O/libperfslice_core.a"
ar rcs "$O/libperfslice_core.a" "$O"/obj/*.o
# Reference C ABI (libperfslice.so) and acceptance binary, built from the
# reference's own sources as they lie.
g++ -std=c++20 -O2 -shared -fPIC -I$R/include -I$R/src -I$O/shim "$R/src/capi.cpp" \
    "$O/libperfslice_core.a" -lpthread -o "$O/libperfslice.so"
g++ -std=c++20 -O2 -I$R/src -I$R/src/core -I$R/tests -I$O/shim "$R/tests/acceptance.cpp" \
    "$O/libperfslice_core.a" -lpthread -o "$O/acceptance" &
# Our harness: golden-vector writer + CPU timing entry points (extern "C").
g++ -std=c++20 -O2 -shared -fPIC -I$R/src -I$R/src/core -I$O/shim "$HERE/ref_harness.cpp" \
    "$O/libperfslice_core.a" -lpthread -o "$O/libps_refharness.so"
wait
echo "build_ref: ok -> $O"
