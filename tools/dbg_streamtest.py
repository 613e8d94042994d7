"""Debug: run the default-stream ordering test with the pre-fix stream argument (handle 0) to
show the test catches the bug (expected: failures)."""
import ctypes as C
import os
import sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import pytest
import paper_2406_03285_b200.rehearsal as R
R._stream_arg = lambda s: C.c_void_p(s.cuda_stream)
sys.exit(pytest.main(["-q", "-m", "gpu", "-k", "default_stream_producer", "tests/test_gpu_run.py"]))
