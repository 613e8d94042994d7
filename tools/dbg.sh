cd $GRAFT_REPO_ROOT
for cfg in "8 3 32 16 6 0" "8 3 32 16 6 1" "4 16 12 8 4 7"; do
  echo "== $cfg" >> gpurun_out/dbg.log
  CUDA_LAUNCH_BLOCKING=1 timeout 60 python tools/debug_parity.py $cfg >> gpurun_out/dbg.log 2>&1
done
CUDA_LAUNCH_BLOCKING=1 timeout 300 python -m pytest tests/test_gpu_engine.py -x -q -k "8-3-32" >> gpurun_out/dbg.log 2>&1
