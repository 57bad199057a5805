#!/usr/bin/env bash
# Round-2 evidence pass: GPU suite, bench (default config, all legs), reference
# arm, launch list, ncu --set full of the three big kernels at configs[1],
# C5 sweep, C3 timing, sparse-path throughput, compute-sanitizer slice.
cd "${GRAFT_REPO_ROOT:-$(pwd)}"; mkdir -p gpurun_out
nvidia-smi --query-gpu=name,memory.total,clocks.sm,clocks.max.sm,power.limit --format=csv > gpurun_out/smi.txt
timeout 1500 python -m pytest tests -m gpu -q -x > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?"; tail -2 gpurun_out/pytest_gpu.log
timeout 900 python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err; echo "bench rc=$?"
timeout 900 python bench.py --impl reference > gpurun_out/bench_ref.json 2> gpurun_out/bench_ref.err; echo "ref rc=$?"
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 60 --csv --log-file gpurun_out/launches.csv \
  python bench.py --steps 2 --warmup 1 --no-e2e --no-cpu-baseline > gpurun_out/b_ncu.log 2>&1; echo "ncu list rc=$?"
bash tools/r2_ncu_c1.sh
bash tools/c5_sweep.sh > gpurun_out/c5_sweep.txt 2>&1; echo "c5 rc=$?"
timeout 600 python tools/c3_units.py > gpurun_out/c3_units.json 2>&1; echo "c3 rc=$?"
timeout 600 python tools/sparse_bench.py 2000 50000 > gpurun_out/sparse_bench.json 2>&1; echo "sparse rc=$?"
SEL="tests/test_gpu_parity.py::test_random_traces_property tests/test_gpu_parity.py::test_full_query_all_parts tests/test_gpu_parity.py::test_auto_anchor_on_device_matches_reference tests/test_gpu_spec.py tests/test_gpu_profiles.py tests/test_gpu_frame.py tests/test_gpu_topology.py tests/test_gpu_units.py::test_units_random_traces tests/test_gpu_units.py::test_units_iterative_equal_unsplit tests/test_gpu_sparse.py" bash tools/r2_sanitize.sh > gpurun_out/sanitize.txt 2>&1; echo "sanitize rc=$?"
