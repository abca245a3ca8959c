"""The C-ABI library (no GPU needed): it builds, loads, exports every symbol
include/gk/gk.h declares, its host-side functions match the oracle bit for
bit, and without a GPU every device entry point fails loudly (no fallback)."""
import ctypes as C
import os
import re
import subprocess
import sys

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(ROOT, "include", "gk", "gk.h")


@pytest.fixture(scope="module")
def libgk():
    from paper_1901_04162_b200 import build
    build.build()
    from paper_1901_04162_b200 import _lib
    return _lib.lib()


def declared_symbols():
    text = open(HEADER).read()
    return sorted(set(re.findall(r"^\s*(?:gk_status|int|uint64_t|void|const char\*)\s+(gk_\w+)\s*\(",
                                 text, re.M)))


def test_header_declares_the_boundary():
    syms = declared_symbols()
    for s in ("gk_table_build", "gk_eval_batch", "gk_fill_rows", "gk_fill_matrix_host",
              "gk_distance_range", "gk_mesh_create", "gk_last_error"):
        assert s in syms


def test_library_exports_every_declared_symbol(libgk):
    out = subprocess.run(["nm", "-D", "--defined-only",
                          os.path.join(ROOT, "paper_1901_04162_b200", "libgk.so")],
                         capture_output=True, text=True, check=True).stdout
    exported = set(re.findall(r" T (gk_\w+)$", out, re.M))
    missing = [s for s in declared_symbols() if s not in exported]
    assert not missing, missing
    from paper_1901_04162_b200._lib import EXPORTS
    assert set(EXPORTS) <= set(declared_symbols())


def test_library_is_sm100a(libgk):
    so = os.path.join(ROOT, "paper_1901_04162_b200", "libgk.so")
    out = subprocess.run(["cuobjdump", "--list-elf", so], capture_output=True, text=True).stdout
    assert "sm_100a" in out


def test_abi_version(libgk):
    assert libgk.gk_abi_version() == 3


def test_host_mesh_generators_match_oracle(libgk, oracle):
    import paper_1901_04162_b200 as gk
    for level in range(0, 4):
        m = gk.generate_sphere_mesh(1.0, level)
        v, t = oracle.sphere_mesh(1.0, level)
        assert np.array_equal(m.vertices, v) and np.array_equal(m.triangles, t)
    mj = gk.jitter(gk.generate_sphere_mesh(1.0, 2), 1901, 1e-3)
    assert np.array_equal(mj.vertices, oracle.jitter(oracle.sphere_mesh(1.0, 2)[0], 1901, 1e-3))
    p = gk.generate_plate_mesh(1.0, 17)
    pv, pt = oracle.plate_mesh(1.0, 17)
    assert np.array_equal(p.vertices, pv) and np.array_equal(p.triangles, pt)
    with pytest.raises(gk.InvalidArgument):
        gk.generate_sphere_mesh(1.0, 7)          # mesh.hpp:156
    with pytest.raises(gk.InvalidArgument):
        gk.generate_sphere_mesh(-1.0, 1)


def test_host_scalars_match_reference_semantics(libgk, oracle):
    import paper_1901_04162_b200 as gk
    assert gk.wavenumber(gk.Medium()) == oracle.wavenumber()
    assert gk.wavenumber(gk.Medium(0.37, 2.3, 1.7)) == oracle.wavenumber(0.37, 2.3, 1.7)
    k = gk.wavenumber(gk.Medium(1.0, 4.0, 1.0, -0.4))
    assert abs(k - 2 * np.pi * np.sqrt(4 - 0.4j)) <= 1e-14 * abs(k)
    assert gk.predicted_calls(320, 4, 3) == 3686400
    with pytest.raises(gk.OverflowErrorGk):
        gk.predicted_calls(1 << 32, 1 << 16, 1 << 16)
    with pytest.raises(gk.InvalidArgument):
        gk.wavenumber(gk.Medium(lambda0=0.0))


def test_device_entry_points_fail_loudly_without_gpu(libgk):
    import torch
    if torch.cuda.is_available():
        pytest.skip("a GPU is present")
    h = C.c_void_p()
    st = libgk.gk_ctx_create(0, C.byref(h))
    assert st == 5 and h.value is None
    assert libgk.gk_last_error()  # a message, not a crash
    import paper_1901_04162_b200 as gk
    with pytest.raises(gk.RuntimeErrorGk):
        gk.Context(0)


def test_package_has_no_cpu_fallback():
    """The product package never imports, links or loads the oracle."""
    pkg = os.path.join(ROOT, "paper_1901_04162_b200")
    banned = ("pyoracle", "liboracle", "gk_oracle", "libgkref", "from oracle", "import oracle")
    for dirpath, _, files in os.walk(pkg):
        for f in files:
            if f.endswith((".py", ".cu", ".cpp", ".h", ".cuh")):
                text = open(os.path.join(dirpath, f)).read()
                assert not any(b in text for b in banned), f


def test_library_does_not_link_nccl(libgk):
    """libgk binds NCCL at first use (dlopen): a DT_NEEDED on the system
    libnccl.so.2 would claim the soname before torch's newer NCCL and break
    `import torch` after the package"""
    out = subprocess.run(["readelf", "-d", os.path.join(ROOT, "paper_1901_04162_b200", "libgk.so")],
                         capture_output=True, text=True, check=True).stdout
    assert "nccl" not in out.lower()
    r = subprocess.run([sys.executable, "-c", "import paper_1901_04162_b200 as gk; "
                        "gk.generate_sphere_mesh(1.0, 1); import torch, torch.distributed; "
                        "print('ok')"], capture_output=True, text=True, cwd=ROOT, timeout=300)
    assert r.returncode == 0 and "ok" in r.stdout, r.stderr[-1500:]
