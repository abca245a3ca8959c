"""fill_rows_gathered (fill + gather fused through CUDA IPC peer memory) with
two processes: a gloo process group for the 64-byte handle broadcast and the
barrier, both ranks on the one GPU (IPC across processes on the same device;
the ranks' kernels never wait on each other).  The gathered matrix on rank 0
equals the single-process fill bit for bit, in both modes."""
import os
import socket

import numpy as np
import pytest

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, out_dir):
    import sys
    sys.path.insert(0, ROOT)
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    import torch
    import torch.distributed as dist
    dist.init_process_group("gloo", rank=rank, world_size=world)
    import paper_1901_04162_b200 as gk
    from paper_1901_04162_b200 import sharding
    mesh = gk.jitter(gk.generate_sphere_mesh(1.0, 2), 1901, 1e-3)
    dm = gk.DeviceMesh(mesh, gk.QuadratureSpec(6, 4))
    lo, hi = sharding.global_distance_range(*dm.distance_range(*sharding.rows_of(rank, world, dm.N)))
    t = gk.DeviceTable(gk.SamplingConfig(r_min=lo, r_max=hi))
    zd, rd = sharding.fill_rows_gathered(dm, gk.Mode.DIRECT, k=2 * np.pi)
    zt, rt = sharding.fill_rows_gathered(dm, gk.Mode.TABLE, table=t)
    calls = torch.tensor([rd.actual_calls + rt.actual_calls], dtype=torch.float64)
    dist.all_reduce(calls)
    if rank == 0:
        ref_d, _ = gk.fill_rows(dm, gk.Mode.DIRECT, k=2 * np.pi)
        ref_t, _ = gk.fill_rows(dm, gk.Mode.TABLE, table=t)
        ok = torch.equal(zd, ref_d) and torch.equal(zt, ref_t)
        ok = ok and int(calls.item()) == 2 * 3 * 6 * 4 * dm.N * (dm.N - 1)
        open(os.path.join(out_dir, "result"), "w").write("ok" if ok else "mismatch")
        del zd, zt
    else:
        assert zd is None and zt is None
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 3])
def test_fused_fill_gather_matches_single_process(tmp_path, world):
    import torch.multiprocessing as mp
    mp.spawn(_worker, args=(world, _port(), str(tmp_path)), nprocs=world, join=True)
    assert (tmp_path / "result").read_text() == "ok"
