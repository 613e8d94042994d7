"""Debug: run a sequence of config_parity cases in one process (argv: python dict literals),
report PASS/FAIL per case."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tests"))
import torch
from test_gpu_configs import config_parity
for a in sys.argv[1:]:
    kw = eval(a)
    env = kw.pop("env", {})
    old = {k: os.environ.get(k) for k in env}
    os.environ.update(env)
    try:
        config_parity(**kw)
        print("PASS", a[:120], flush=True)
    except AssertionError as e:
        print("FAIL", a[:120], str(e)[:600], flush=True)
    for k, v in old.items():
        if v is None:
            os.environ.pop(k, None)
        else:
            os.environ[k] = v
