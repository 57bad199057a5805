#!/usr/bin/env bash
# One GPU-box pass: environment probe, GPU parity tests, bench (small + full),
# ncu launch list and one full capture of the fused kernel.  Outputs land in
# gpurun_out/ (merged back by gpurun).
set -u
cd "${GRAFT_REPO_ROOT:-$(pwd)}"
mkdir -p gpurun_out
STAGES="${STAGES:-probe tests bench_small bench ncu_list ncu_full}"
for s in $STAGES; do
  echo "=== $s $(date +%T)"
  case $s in
    probe) { nvidia-smi; free -g; nproc; lscpu | head -20; df -h /dev/shm /tmp; } > gpurun_out/probe.txt 2>&1 ;;
    tests) timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" ;;
    bench_small) timeout 600 python bench.py --traces 10000 --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/bench_10k.log 2>&1; echo "rc=$?"; tail -c 3000 gpurun_out/bench_10k.log ;;
    bench) timeout 1500 python bench.py > gpurun_out/bench_full.log 2>&1; echo "rc=$?"; tail -c 3000 gpurun_out/bench_full.log ;;
    bench_ref) timeout 900 python bench.py --impl reference > gpurun_out/bench_ref.log 2>&1; echo "rc=$?"; tail -c 2000 gpurun_out/bench_ref.log ;;
    ncu_list) timeout 1200 ncu --metrics gpu__time_duration.sum --clock-control none --csv \
        --log-file gpurun_out/launches.csv python bench.py --steps 2 --warmup 1 --no-e2e --no-cpu-baseline \
        > gpurun_out/ncu_list.log 2>&1; echo "rc=$?"; tail -5 gpurun_out/ncu_list.log ;;
    ncu_full) timeout 1200 ncu --set full --clock-control none --import-source on -k regex:k_trace_query \
        -s 1 -c 1 -f -o gpurun_out/prof_trace_query python bench.py --traces 10000 --steps 1 --warmup 1 --no-e2e \
        --no-cpu-baseline > gpurun_out/ncu_full.log 2>&1; echo "rc=$?"; tail -5 gpurun_out/ncu_full.log ;;
  esac
done
echo "=== done $(date +%T)"
