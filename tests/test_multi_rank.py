"""The N > 1 path (paper_1901_04162_b200.sharding, used by bench.py) on CPU
(gloo, world_size 2 and 3), with the oracle as the per-rank compute: each rank
takes rows_of(rank, world, N), computes its K1 distance range, one 16-byte
all-reduce (global_distance_range) gives the global range, every rank builds
the identical plan from it, fills its own rows, gather_rows collects the
blocks on rank 0, and the result equals the single-process fill bit for bit
(the GPU-side union property is tests/test_gpu_fill.py)."""
import math
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, out_dir):
    import sys
    sys.path.insert(0, ROOT)
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from paper_1901_04162_b200 import sharding
    from oracle.pyoracle import DIRECT, TABLE, Oracle, SamplingConfig
    o = Oracle()
    v, t = o.sphere_mesh(1.0, 1)
    v = o.jitter(v, 1901, 1e-3)
    N = t.shape[0]
    rb, re = sharding.rows_of(rank, world, N)
    lo, hi = o.distance_range(v, t, 6, 4, rb, re)
    glo, ghi = sharding.global_distance_range(lo, hi)
    plan = o.build_plan(SamplingConfig(r_min=glo, r_max=ghi, samples_per_wavelength=2000))
    digest = torch.tensor([float(plan.abscissae.size), float(plan.abscissae.sum())],
                          dtype=torch.float64)
    digests = [torch.zeros(2, dtype=torch.float64) for _ in range(world)]
    dist.all_gather(digests, digest)
    ev = o.evaluator(plan, 2 * math.pi)
    zt, rept = o.fill_rows(v, t, 6, 4, TABLE, 2 * math.pi, ev=ev, row_begin=rb, row_end=re)
    zd, repd = o.fill_rows(v, t, 6, 4, DIRECT, 2 * math.pi, row_begin=rb, row_end=re)
    full = sharding.gather_rows(torch.from_numpy(zd), N, dst=0)
    if rank == 0:
        np.save(os.path.join(out_dir, "gathered.npy"), full.numpy())
    else:
        assert full is None
    np.savez(os.path.join(out_dir, f"rank{rank}.npz"), zt=zt, zd=zd, rb=rb, re=re, lo=glo, hi=ghi,
             digests=torch.stack(digests).numpy(), calls=rept.actual_calls,
             fb=rept.fallback_calls)
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 3])
def test_row_sharding_matches_single_process(tmp_path, oracle, world):
    mp.spawn(_worker, args=(world, _free_port(), str(tmp_path)), nprocs=world, join=True)
    parts = [np.load(tmp_path / f"rank{r}.npz") for r in range(world)]
    v, t = oracle.sphere_mesh(1.0, 1)
    v = oracle.jitter(v, 1901, 1e-3)
    N = t.shape[0]
    lo, hi = oracle.distance_range(v, t, 6, 4)
    for p in parts:   # the all-reduced range is the global one, on every rank
        assert float(p["lo"]) == lo and float(p["hi"]) == hi
        assert np.array_equal(p["digests"][0], p["digests"][1])  # identical tables
    assert int(parts[0]["rb"]) == 0 and int(parts[-1]["re"]) == N
    for a, b in zip(parts[:-1], parts[1:]):
        assert int(a["re"]) == int(b["rb"])
    from oracle.pyoracle import DIRECT, TABLE, SamplingConfig
    plan = oracle.build_plan(SamplingConfig(r_min=lo, r_max=hi, samples_per_wavelength=2000))
    ev = oracle.evaluator(plan, 2 * math.pi)
    zt, _ = oracle.fill_rows(v, t, 6, 4, TABLE, 2 * math.pi, ev=ev, threads=4)
    zd, _ = oracle.fill_rows(v, t, 6, 4, DIRECT, 2 * math.pi, threads=4)
    assert np.array_equal(np.concatenate([p["zt"] for p in parts]), zt)
    assert np.array_equal(np.concatenate([p["zd"] for p in parts]), zd)
    assert np.array_equal(np.load(tmp_path / "gathered.npy"), zd)   # gather_rows on rank 0
    assert sum(int(p["calls"]) for p in parts) == 3 * 6 * 4 * N * (N - 1)
    assert all(int(p["fb"]) == 0 for p in parts)


@pytest.mark.parametrize("world,N", [(1, 1280), (2, 1280), (8, 81920), (3, 80), (8, 20)])
def test_rows_of_partitions_exactly(world, N):
    import bench
    blocks = [bench.rows_of(r, world, N) for r in range(world)]
    covered = [i for b, e in blocks for i in range(b, e)]
    assert covered == list(range(N))
    chunk = (N + world - 1) // world    # matfill.hpp:211-215
    assert all(e - b <= chunk for b, e in blocks)


@pytest.mark.parametrize("world,N", [(1, 1280), (2, 1280), (8, 81920), (3, 80), (8, 20), (7, 5),
                                     (5, 0)])
def test_c_abi_rows_of_is_the_reference_chunking(world, N):
    """gk_rows_of (host-only C ABI, used by gk_fill_sharded / gk_gather_rows)
    gives the reference's chunks, chunk = ceil(N / threads) (matfill.hpp:211-215)"""
    from paper_1901_04162_b200 import sharding
    import bench
    chunk = (N + world - 1) // world
    for r in range(world):
        b, e = sharding.rows_of(r, world, N)
        assert (b, e) == bench.rows_of(r, world, N) == (min(N, r * chunk), min(N, r * chunk + chunk))


def test_c_abi_comm_rejects_bad_arguments_without_a_device():
    """the communicator entry points fail with a status (no crash) on bad
    arguments; gk_rows_of validates its ranks"""
    import ctypes as C
    from paper_1901_04162_b200._lib import lib
    L = lib()
    b, e = C.c_uint64(), C.c_uint64()
    assert L.gk_rows_of(10, 0, 0, C.byref(b), C.byref(e)) == 1
    assert L.gk_rows_of(10, 2, 2, C.byref(b), C.byref(e)) == 1
    assert L.gk_comm_init(None, None, 1, 0, None) == 1
    assert L.gk_comm_init_all(None, 0, None) == 1
    assert L.gk_gather_rows(None, None, None, 10, 0, None) == 1
    assert L.gk_comm_destroy(None) == 0
