C="dict(K=100,cap=6,T=4,c=14,steps=100,S=301056,b=128,r=28,N=4)"
echo "== multi"; timeout 300 python tools/dbg_cfg.py "$C" "$C" "$C" 2>&1 | grep -v Warn | cut -c1-6,120-900
T="python -m torch.distributed.run --nnodes=1 --master-addr 127.0.0.1 --master-port 29512"
for n in 1 2 4; do echo "== timeline N=$n"; timeout 200 $T --nproc-per-node $n tools/mp_persist_timeline.py c2 300 2>&1 | grep -v Warn | tail -25; done
