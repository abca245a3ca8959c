"""The C++ drop-in adapter (include/gk/gk.hpp) driven from a C++ host
program on the B200 (tests/cpp/test_adapter.cpp)."""
import subprocess

import pytest

pytestmark = pytest.mark.gpu


def test_cpp_adapter_program(gk):
    from paper_1901_04162_b200.build import build_cpp_test
    exe = build_cpp_test()
    r = subprocess.run([exe], capture_output=True, text=True, timeout=300)
    assert r.returncode == 0, r.stdout + r.stderr
    assert "ALL OK" in r.stdout
