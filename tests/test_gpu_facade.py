"""The C++ facade (include/drb_rb.hpp) driven from a C++ program: KATs, usage errors and 60
engine iterations bit-exact against the C oracle (tests/cpp/facade_parity.cpp)."""
import os
import subprocess

import pytest

pytestmark = pytest.mark.gpu

EXE = os.path.join(os.path.dirname(__file__), "cpp", "facade_parity")


def test_cpp_facade_parity():
    assert os.path.exists(EXE), "build first: python -c 'import __graft_entry__ as g; g.build()'"
    res = subprocess.run([EXE], capture_output=True, text=True, timeout=120)
    assert res.returncode == 0, res.stdout + res.stderr
    assert "bit-exact" in res.stdout


def test_cpp_input_facade_parity():
    exe = os.path.join(os.path.dirname(__file__), "cpp", "input_parity")
    assert os.path.exists(exe), "build first: python -c 'import __graft_entry__ as g; g.build()'"
    gold = os.path.join(os.path.dirname(__file__), "golden")
    res = subprocess.run([exe, gold], capture_output=True, text=True, timeout=120)
    assert res.returncode == 0, res.stdout + res.stderr
    assert "bit-exact" in res.stdout
