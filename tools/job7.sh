cd $GRAFT_REPO_ROOT
timeout 900 python -m pytest tests -x -q -m gpu > gpurun_out/pytest_cnt2.log 2>&1; echo "pytest rc $?"; tail -3 gpurun_out/pytest_cnt2.log
STEPS=10000 bash tools/ab_bench.sh "tools/ablib/libdrb_cnt.so tools/ablib/libdrb_cnt2.so"
