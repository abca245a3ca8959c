"""Row-block sharding of the fill across ranks.

The reference parallelises fill_matrix over std::threads, each taking a
contiguous chunk of observation rows, chunk = ceil(N / threads)
(matfill.hpp:206-221); entries are independent, so results do not depend on
the thread count.  Here the same chunking runs one rank per GPU:

1. every rank computes the pair-distance range of its own rows (K1),
2. ONE 16-byte all-reduce (MIN of {r_min, -r_max}) makes it global,
3. every rank builds the identical table from the global range (the device
   build is deterministic) and fills its rows -- no data-path collective,
4. optionally the row blocks are gathered to one rank: point-to-point sends
   into the destination's row slices after the fill (gather_rows), or fused
   with it -- every rank's fill kernel storing straight into the destination
   rank's matrix through CUDA IPC peer memory (fill_rows_gathered).

The GPU path lives in C++ behind the C ABI (csrc/comm.cu): a ``Comm`` is
libgk's own NCCL communicator, and ``distance_range_global``,
``fill_rows_sharded`` and ``gather_rows_nccl`` are thin wrappers of
gk_distance_range_global / gk_fill_sharded / gk_gather_rows -- a C++ caller
of the reference gets the same sharded fill without Python
(tools/gk_sharded_fill.cpp).  torch.distributed only ships the 128-byte
NCCL id here.  The torch.distributed helpers below (global_distance_range,
gather_rows) are the same steps over any backend: gloo on CPU for the
multi-rank tests.
"""
from __future__ import annotations

import ctypes as C


def rows_of(rank: int, world: int, N: int) -> tuple[int, int]:
    """Contiguous row block [begin, end) of `rank` (matfill.hpp:211-215):
    gk_rows_of, the partition the C++ sharded fill uses (host-only)."""
    from ._lib import check, lib
    b, e = C.c_uint64(), C.c_uint64()
    check(lib().gk_rows_of(N, world, rank, C.byref(b), C.byref(e)), "rows_of")
    return b.value, e.value


class Comm:
    """gk_comm: libgk's NCCL communicator on one context's device (C++,
    csrc/comm.cu).  Made collectively: rank 0 creates the 128-byte id
    (gk_comm_unique_id), the id travels over the torch.distributed group
    (any transport would do), every rank calls gk_comm_init."""

    def __init__(self, ctx, group=None):
        import torch
        import torch.distributed as dist

        from ._lib import check, lib
        self.ctx = ctx
        if dist.is_available() and dist.is_initialized():
            nranks, rank = dist.get_world_size(group), dist.get_rank(group)
        else:
            nranks, rank = 1, 0
        idb = (C.c_ubyte * 128)()
        if rank == 0:
            check(lib().gk_comm_unique_id(idb), "gk_comm_unique_id")
        if nranks > 1:
            on_dev = dist.get_backend(group) == "nccl"
            t = torch.tensor(list(bytes(idb)), dtype=torch.uint8,
                             device=f"cuda:{ctx.device}" if on_dev else "cpu")
            dist.broadcast(t, src=dist.get_global_rank(group, 0) if group else 0, group=group)
            idb = (C.c_ubyte * 128).from_buffer_copy(bytes(t.cpu().tolist()))
        h = C.c_void_p()
        check(lib().gk_comm_init(ctx.h, idb, nranks, rank, C.byref(h)), "gk_comm_init")
        self.h, self.nranks, self.rank = h, nranks, rank

    def info(self) -> tuple[int, int]:
        """(nranks, rank) as the NCCL communicator reports them"""
        from ._lib import check, lib
        n, r = C.c_int(), C.c_int()
        check(lib().gk_comm_info(self.h, C.byref(n), C.byref(r)), "gk_comm_info")
        return n.value, r.value

    def __del__(self):
        from . import _lib
        h = getattr(self, "h", None)
        if h and _lib._lib is not None:
            try:
                _lib._lib.gk_comm_destroy(h)
            except Exception:  # interpreter shutdown
                pass
            self.h = None


def distance_range_global(comm: Comm, dmesh) -> tuple[float, float]:
    """K1 over this rank's rows + the 16-byte NCCL MIN all-reduce, on the
    device (gk_distance_range_global)"""
    from ._lib import check, lib
    comm.ctx.bind_stream()
    lo, hi = C.c_double(), C.c_double()
    check(lib().gk_distance_range_global(comm.ctx.h, comm.h, dmesh.h, C.byref(lo), C.byref(hi)),
          "distance_range_global")
    return lo.value, hi.value


def fill_rows_sharded(comm: Comm, dmesh, mode, out, cfg=None, medium=None, kind=None,
                      options=None, report: bool = True):
    """This rank's share of the fill (gk_fill_sharded): rows rows_of(rank)
    into `out` (a CUDA complex128 (rows, >= N) view); TABLE with cfg.r_min or
    cfg.r_max <= 0 takes the global K1 range.  Returns (FillReport | None,
    (r_min, r_max) of the table or None)."""
    from . import gktab
    from ._lib import FillReportC, check, lib
    kind = gktab.KernelKind.GreenOverR if kind is None else kind
    medium = medium or gktab.Medium()
    rb, re = rows_of(comm.rank, comm.nranks, dmesh.N)
    rep = FillReportC()
    rng = (C.c_double * 2)()
    comm.ctx.bind_stream()
    check(lib().gk_fill_sharded(comm.ctx.h, comm.h, dmesh.h, int(mode),
                                C.byref(cfg.c()) if cfg is not None else None,
                                C.byref(medium.c()), int(kind),
                                out.data_ptr() if re > rb else None,
                                out.stride(0) if re > rb else dmesh.N,
                                C.byref(options.c()) if options is not None else None,
                                C.byref(rep) if report else None, rng), "fill_matrix")
    return (gktab.FillReport.from_c(rep) if report else None,
            (rng[0], rng[1]) if int(mode) == int(gktab.Mode.TABLE) else None)


def gather_rows_nccl(comm: Comm, z_local, N: int, root: int = 0, out=None):
    """Every rank's row block into root's N x N device matrix (gk_gather_rows:
    grouped ncclSend / ncclRecv, no staging).  Returns `out` on root."""
    import torch

    from ._lib import check, lib
    rb, re = rows_of(comm.rank, comm.nranks, N)
    if comm.rank == root and out is None:
        out = torch.empty((N, N), dtype=torch.complex128, device=f"cuda:{comm.ctx.device}")
    comm.ctx.bind_stream()
    check(lib().gk_gather_rows(comm.ctx.h, comm.h,
                               z_local.data_ptr() if re > rb else None, N, root,
                               out.data_ptr() if comm.rank == root else None),
          "gather_rows")
    return out if comm.rank == root else None


def global_distance_range(lo: float, hi: float, device=None, group=None) -> tuple[float, float]:
    """All-reduce of the per-rank range: one MIN over the 16-byte {lo, -hi}.

    Ranks with no rows pass (inf, 0)."""
    import torch
    import torch.distributed as dist
    if not (dist.is_available() and dist.is_initialized()) or dist.get_world_size(group) == 1:
        return lo, hi
    t = torch.tensor([lo, -hi], dtype=torch.float64, device=device)
    dist.all_reduce(t, op=dist.ReduceOp.MIN, group=group)
    return float(t[0]), -float(t[1])


def gather_rows(z_local, N: int, dst: int = 0, out=None, group=None):
    """Gather every rank's row block of Z into an N x N matrix on rank `dst`.

    `z_local` holds this rank's rows (rows_of(rank, world, N)) with N columns
    (row-major, contiguous).  On `dst` the result is `out` (allocated like
    z_local when None) with z_local copied into its own slice unless it
    already is that slice; other ranks return None.  Every block lands
    directly in its contiguous row slice of `out` (no staging copy)."""
    import torch
    import torch.distributed as dist
    world = dist.get_world_size(group)
    rank = dist.get_rank(group)
    rb, re = rows_of(rank, world, N)
    if z_local.shape[0] < re - rb or (re > rb and z_local.shape[1] != N):
        raise ValueError("gather_rows: z_local must hold this rank's rows x N columns")
    if rank != dst:
        if re > rb:
            dist.send(z_local[: re - rb].contiguous(), dst=dst, group=group)
        return None
    if out is None:
        out = torch.empty((N, N), dtype=z_local.dtype, device=z_local.device)
    own = out[rb:re]
    if re > rb and own.data_ptr() != z_local.data_ptr():
        own.copy_(z_local[: re - rb])
    reqs = []
    for r in range(world):
        b, e = rows_of(r, world, N)
        if r != dst and e > b:
            reqs.append(dist.irecv(out[b:e], src=r, group=group))
    for q in reqs:
        q.wait()
    return out


class _DeviceMatrix:
    """__cuda_array_interface__ view of raw device memory (torch.as_tensor
    keeps this object alive while the tensor lives; `release` runs after)."""

    def __init__(self, ptr: int, shape, release=None):
        self.__cuda_array_interface__ = {"shape": tuple(shape), "typestr": "<c16",
                                         "data": (ptr, False), "version": 3, "strides": None}
        self._release = release

    def __del__(self):
        if self._release is not None:
            try:
                self._release()
            except Exception:  # interpreter shutdown
                pass


def fill_rows_gathered(dmesh, mode, kind=None, table=None, k: complex = 0.0, dst: int = 0,
                       group=None):
    """Fill and gather fused (SURVEY 8e step 5 without a separate collective):
    rank `dst` allocates the full N x N matrix as shareable device memory
    (gk_shared_alloc), its 64-byte IPC handle is broadcast over the process
    group, every other rank maps it (gk_ipc_open), and each rank's fill kernel
    stores its row block rows_of(rank, world, N) straight into it -- NVLink
    peer stores between the GPUs of one node, overlapped with the compute by
    construction.  Returns (Z, report) on `dst` (Z a complex128 CUDA tensor
    owning the allocation) and (None, report) elsewhere."""
    import ctypes as C

    import torch
    import torch.distributed as dist

    from . import gktab
    from ._lib import check, lib

    kind = gktab.KernelKind.GreenOverR if kind is None else kind
    ctx = dmesh.ctx
    N = dmesh.N
    world = dist.get_world_size(group)
    rank = dist.get_rank(group)
    rb, re = rows_of(rank, world, N)
    handle = (C.c_ubyte * 64)()
    ptr = C.c_void_p()
    if rank == dst:
        check(lib().gk_shared_alloc(ctx.h, N * N * 16, C.byref(ptr), handle), "gk_shared_alloc")
    on_dev = dist.get_backend(group) == "nccl"
    ht = torch.tensor(list(bytes(handle)), dtype=torch.uint8,
                      device=f"cuda:{ctx.device}" if on_dev else "cpu")
    dist.broadcast(ht, src=dst, group=group)
    if rank != dst:
        handle = (C.c_ubyte * 64).from_buffer_copy(bytes(ht.cpu().tolist()))
        check(lib().gk_ipc_open(ctx.h, handle, C.byref(ptr)), "gk_ipc_open")
    h, p = ctx.h, ptr.value
    # the closure holds the Context itself: it must outlive the allocation
    release = (lambda c=ctx: lib().gk_shared_free(c.h, C.c_void_p(p))) if rank == dst else None
    # no device= here: the mapped memory lives on dst's GPU and torch must take
    # the device from the pointer -- asking for this rank's device would make
    # it copy the matrix instead of viewing the peer memory
    full = torch.as_tensor(_DeviceMatrix(p, (N, N), release))
    assert full.data_ptr() == p, "fill_rows_gathered: the matrix must be a view, not a copy"
    rep = None
    try:
        if re > rb:
            _, rep = gktab.fill_rows(dmesh, mode, kind=kind, table=table, k=k, row_begin=rb,
                                     row_end=re, out=full[rb:re])
        ctx.synchronize()
        dist.barrier(group)   # every block has landed in dst's matrix
    finally:
        if rank != dst:
            del full
            check(lib().gk_ipc_close(h, C.c_void_p(p)), "gk_ipc_close")
    return (full if rank == dst else None), rep


def shard_summary(world: int, N: int) -> list[tuple[int, int]]:
    """All row blocks, rank order (for reports)."""
    return [rows_of(r, world, N) for r in range(world)]


def evals_of_rows(rows: int, N: int, m: int, n: int) -> int:
    """actual_calls of a row block: 3 m n rows (N - 1) (matfill.hpp:200)."""
    return 3 * m * n * rows * (N - 1) if N > 0 else 0


__all__ = ["rows_of", "Comm", "distance_range_global", "fill_rows_sharded", "gather_rows_nccl",
           "global_distance_range", "gather_rows", "fill_rows_gathered", "shard_summary",
           "evals_of_rows"]
