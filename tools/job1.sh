cd $GRAFT_REPO_ROOT
timeout 900 python -m pytest tests -x -q -m gpu > gpurun_out/pytest_noinst.log 2>&1; echo "pytest rc $?"
tail -2 gpurun_out/pytest_noinst.log
timeout 600 ncu --set full --import-source on --clock-control none -k regex:drb_run_kernel --launch-skip 8 -c 1 -o gpurun_out/ncu_run_noinst -f python bench.py --steps 200 --warmup 5 --no-cpu --e2e-steps 10 > gpurun_out/ncu_run_noinst.log 2>&1; echo "ncu rc $?"
