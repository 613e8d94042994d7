set -x
mkdir -p gpurun_out
python -m pytest tests -m gpu -x -q 2>&1 | tail -5
python bench.py --no-cpu > gpurun_out/b1.json 2>gpurun_out/b1.err; tail -1 gpurun_out/b1.json
python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29511 bench.py --gpus 2 --no-cpu > gpurun_out/b2.json 2>gpurun_out/b2.err; tail -1 gpurun_out/b2.json
