P="dict(K=1000,cap=2,S=150528,b=56,c=14,r=7,T=1,steps=400,slab_check=True,post_steps=False)"
DRB_DBG=17408 timeout 600 python tools/dbg_seq.py "dict(K=10,cap=2,S=1024,b=56,c=14,r=7,T=1,steps=10,post_steps=False)" "$P" "$P" "$P" 2>&1 | grep -v Warn | cut -c1-200
C="dict(K=100,cap=6,T=4,c=14,steps=100,S=301056,b=128,r=28,N=4)"
timeout 300 python tools/dbg_seq.py "$C" "$C" "$C" 2>&1 | grep -v Warn | cut -c1-200
timeout 1200 python -m pytest tests -m gpu -q > gpurun_out/pytest_all.log 2>&1; echo pytest_rc=$?; tail -3 gpurun_out/pytest_all.log
