cd $GRAFT_REPO_ROOT
timeout 900 python -m pytest tests -x -q -m gpu > gpurun_out/pytest_spec.log 2>&1; echo "pytest rc $?"; tail -2 gpurun_out/pytest_spec.log
DBGS="0 128" bash tools/ab_bench.sh "tools/ablib/libdrb_noinst.so tools/ablib/libdrb_spec.so"
