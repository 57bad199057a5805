cd ${GRAFT_REPO_ROOT}
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/pytest_gpu.log
for v in base build/variants/nocrosstma.so; do if [ $v = base ]; then unset PSG_LIB; else export PSG_LIB=$v; fi; echo "== $v"; python tools/timeline.py 100000; done
unset PSG_LIB
STAGES=ncu_list bash tools/gpu_round.sh > /dev/null 2>&1
