"""The multi-GPU fill behind the C ABI (csrc/comm.cu) on the one
GPU a test box has: libgk's own NCCL communicator with one rank (NCCL refuses
two ranks on one device, so the N-rank exchange itself is exercised by the
CPU gloo tests, tests/test_multi_rank.py, and on multi-GPU nodes by bench.py
--gpus N and tools/gk_sharded_fill).  Checked here: the communicator, the
device-side 16-byte MIN all-reduce of the range, gk_fill_sharded and
gk_gather_rows reproduce the single-GPU results bit for bit, from Python and
from the C++ driver."""
import json
import subprocess

import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def sphere(gk, level):
    return gk.jitter(gk.generate_sphere_mesh(1.0, level), 1901, 1e-3)


def test_comm_one_rank_range_fill_gather(gk):
    import torch
    from paper_1901_04162_b200 import sharding
    ctx = gk.Context.get(0)
    comm = sharding.Comm(ctx)
    assert comm.info() == (1, 0)
    dm = gk.DeviceMesh(sphere(gk, 3), gk.QuadratureSpec(6, 4))
    # the all-reduced range of a single rank is gk_distance_range's, bitwise
    assert sharding.distance_range_global(comm, dm) == dm.distance_range()
    N = dm.N
    med = gk.Medium(lambda0=0.5)
    for mode in (gk.Mode.DIRECT, gk.Mode.TABLE):
        z = torch.empty((N, N), dtype=torch.complex128, device="cuda:0")
        cfg = gk.SamplingConfig(r_min=0.0, r_max=0.0, samples_per_wavelength=2000)
        rep, rng = sharding.fill_rows_sharded(comm, dm, mode, z, cfg=cfg, medium=med)
        if mode == gk.Mode.TABLE:
            assert rng == dm.distance_range()
            t = gk.DeviceTable(gk.SamplingConfig(r_min=rng[0], r_max=rng[1],
                                                 samples_per_wavelength=2000), med)
            ref, rref = gk.fill_rows(dm, mode, table=t)
        else:
            ref, rref = gk.fill_rows(dm, mode, k=gk.wavenumber(med))
        assert torch.equal(z, ref)
        assert rep.actual_calls == rref.actual_calls and rep.fallback_calls == rref.fallback_calls
        full = sharding.gather_rows_nccl(comm, z, N, root=0)
        assert torch.equal(full, ref)


@pytest.mark.parametrize("mode", ["direct", "table"])
def test_cpp_sharded_fill_driver(gk, mode):
    """tools/gk_sharded_fill: the C++-only multi-GPU driver (gk_comm_init_all,
    one host thread per GPU) with the one GPU here: gathered Z bitwise equal to
    a plain one-GPU fill, NCCL reports the expected rank count"""
    from paper_1901_04162_b200.build import build_tools
    exe = build_tools()
    r = subprocess.run([exe, "--gpus", "1", "--level", "3", "--lambda", "0.5", "--mode", mode,
                        "--S", "2000", "--reps", "2", "--check", "1"],
                       capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stdout + r.stderr
    d = json.loads([ln for ln in r.stdout.splitlines() if ln.startswith("{")][-1])
    assert d["n_gpus"] == 1 and d["N"] == 1280 and d["nccl_nranks_ok"]
    assert d["bitwise_equal_to_one_gpu"] is True and d["gathered"]
    assert d["actual_calls"] == 3 * 6 * 4 * 1280 * 1279 and d["fill_ms_max_over_ranks"] > 0
