cd "${GRAFT_REPO_ROOT:-$(pwd)}"; mkdir -p gpurun_out
PSG_TRACE_QUERY=1 timeout 900 python -m pytest tests/test_gpu_spec.py -q -x > gpurun_out/pytest_spec.log 2>&1; echo "spec rc=$?"; tail -3 gpurun_out/pytest_spec.log
VARIANTS="ov2:PSG_OVERLAP=2 ov4:PSG_OVERLAP=4 nospec:PSG_NO_SPEC=1" REPS=2 bash tools/ab_env.sh
