"""The raw C ABI under bad arguments: every entry point returns a status code
(GK_ERR_INVALID_ARGUMENT = 1, ...) with a message in gk_last_error -- no crash,
no device fault -- and the context keeps working afterwards."""
import ctypes as C

import numpy as np
import pytest

pytestmark = pytest.mark.gpu
INVALID = 1


def test_abi_rejects_bad_arguments(gk):
    from paper_1901_04162_b200._lib import lib
    L = lib()
    ctx = gk.Context.get(0)
    h = ctx.h
    mesh = gk.generate_sphere_mesh(0.5, 1)
    dm = gk.DeviceMesh(mesh, gk.QuadratureSpec(4, 3))
    t = gk.DeviceTable(gk.SamplingConfig())
    N = dm.N
    calls = [
        lambda: L.gk_fill_rows(None, dm.h, 0, None, 1, 1.0, 0.0, 0, N, None, N, None, None),   # null ctx
        lambda: L.gk_fill_rows(h, None, 0, None, 1, 1.0, 0.0, 0, N, None, N, None, None),      # null mesh
        lambda: L.gk_fill_rows(h, dm.h, 7, None, 1, 1.0, 0.0, 0, N, None, N, None, None),      # bad mode
        lambda: L.gk_fill_rows(h, dm.h, 0, None, 5, 1.0, 0.0, 0, N, None, N, None, None),      # bad kind
        lambda: L.gk_fill_rows(h, dm.h, 0, None, 1, 1.0, 0.0, 5, 2, None, N, None, None),      # rows
        lambda: L.gk_fill_rows(h, dm.h, 0, None, 1, 1.0, 0.0, 0, N, None, N - 1, None, None),  # ldz
        lambda: L.gk_fill_rows(h, dm.h, 0, None, 1, 1.0, 0.0, 0, N, None, N, None, None),      # null z
        lambda: L.gk_fill_rows(h, dm.h, 1, None, 1, 1.0, 0.0, 0, 0, None, N, None, None),      # no table
        lambda: L.gk_fill_rows(h, dm.h, 0, None, 1, -1.0, 0.0, 0, 0, None, N, None, None),     # k < 0
        lambda: L.gk_eval_batch(h, None, 1, 1.0, 0.0, None, 10, None, None),             # null buf
        lambda: L.gk_locate(h, None, None, 0, None),                                      # no table
        lambda: L.gk_table_build(h, None, None, 3, None),
        lambda: L.gk_table_build(h, C.byref(t.cfg.c()), C.byref(gk.Medium().c()), 0,
                                 C.byref(C.c_void_p())),                                  # degree 0
        lambda: L.gk_table_build(h, C.byref(t.cfg.c()), C.byref(gk.Medium().c()), 9,
                                 C.byref(C.c_void_p())),                                  # degree 9
        lambda: L.gk_mesh_create(h, None, 3, None, 1, 4, 3, C.byref(C.c_void_p())),      # null data
        lambda: L.gk_error_sweep(h, t.h, 1, 1, 0, None),                                 # 0 probes
        lambda: L.gk_compare_fills(h, None, None, 3, 3, 0, 2, None, None),               # ld < N
        lambda: L.gk_accumulate_batch(h, None, 1, 1.0, 0.0, None, None, 4, 2, None, None),
        lambda: L.gk_distance_range(h, dm.h, 5, 2, None, None),
        lambda: L.gk_shared_alloc(h, 0, None, None),
        lambda: L.gk_rows_of(10, 0, 0, None, None),                                      # nranks
        lambda: L.gk_comm_init(h, None, 1, 0, None),                                      # null id
        lambda: L.gk_comm_init_all(None, 1, None),
        lambda: L.gk_gather_rows(h, None, None, N, 0, None),                              # no comm
        lambda: L.gk_distance_range_global(h, None, dm.h, None, None),
        lambda: L.gk_fill_sharded(h, None, dm.h, 0, None, None, 1, None, N, None, None, None),
    ]
    for i, call in enumerate(calls):
        st = call()
        assert st != 0, i
        assert L.gk_last_error(), i
    # the context still works
    z, rep = gk.fill_rows(dm, gk.Mode.DIRECT, k=2 * np.pi)
    assert rep.actual_calls == 3 * 4 * 3 * N * (N - 1)
