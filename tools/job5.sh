cd $GRAFT_REPO_ROOT
timeout 900 python -m pytest tests -x -q -m gpu > gpurun_out/pytest_cnt.log 2>&1; echo "pytest rc $?"; tail -3 gpurun_out/pytest_cnt.log
bash tools/ab_bench.sh "tools/ablib/libdrb_arrw.so tools/ablib/libdrb_cnt.so"
