"""Debug: tests/test_gpu_configs.config_parity over a parameter grid; prints PASS/FAIL per case."""
import os, sys, traceback
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tests"))
os.environ.setdefault("DRB_TIMEOUT_MS", "5000")
import gc
import torch
from test_gpu_configs import config_parity
cases = [eval(a) for a in sys.argv[1:]]
for cs in cases:
    if os.environ.get("DBG_GC"):
        gc.collect()
    kw = dict(cs)
    try:
        config_parity(**kw)
        print("PASS", kw, flush=True)
    except AssertionError as e:
        print("FAIL", kw, str(e).splitlines()[0][:300], flush=True)
    except Exception as e:
        print("ERR", kw, type(e).__name__, str(e)[:300], flush=True)
