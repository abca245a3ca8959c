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


def test_device_kernel_plugs_into_reference_fill_matrix(gk):
    """gk::DeviceTableKernel at the reference's own plugin seam: the unmodified
    gktab::fill_matrix driven by it vs by the reference's TableKernel on the
    same plan (oracle/_ref/plug, built from tests/cpp/plug_into_reference.cpp)."""
    import os
    import subprocess
    exe = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))),
                       "oracle", "_ref", "plug")
    if not os.path.exists(exe):
        import pytest
        pytest.skip("oracle/_ref/plug not built (reference tree absent at build time)")
    r = subprocess.run([exe], capture_output=True, text=True, timeout=600)
    assert r.returncode == 0 and "-> OK" in r.stdout, r.stdout + r.stderr
