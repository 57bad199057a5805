#!/usr/bin/env bash
# compute-sanitizer memcheck + racecheck over a representative slice of the GPU
# suite (every kernel family: generator, loaders, pass 1/2, layout, stats,
# outliers, topology, profiles, frame, anchor).  Logs to gpurun_out/.
cd "${GRAFT_REPO_ROOT:-$(pwd)}"; mkdir -p gpurun_out
SEL=${SEL:-"tests/test_gpu_parity.py::test_random_traces_property tests/test_gpu_parity.py::test_full_query_all_parts tests/test_gpu_parity.py::test_auto_anchor_on_device_matches_reference tests/test_gpu_spec.py tests/test_gpu_profiles.py tests/test_gpu_frame.py tests/test_gpu_topology.py"}
for tool in memcheck racecheck; do
  timeout ${SAN_TIMEOUT:-1500} compute-sanitizer --tool $tool --target-processes all --error-exitcode 99 \
    --log-file gpurun_out/sanitizer_$tool.%p.log \
    python -m pytest $SEL -q -x -k "one" > gpurun_out/sanitizer_${tool}_pytest.log 2>&1
  echo "$tool rc=$?"; tail -2 gpurun_out/sanitizer_${tool}_pytest.log
done
grep -h "ERROR SUMMARY" gpurun_out/sanitizer_*.log | sort | uniq -c
