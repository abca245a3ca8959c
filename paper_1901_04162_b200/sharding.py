"""Row-block sharding of the fill across ranks.

The reference parallelises fill_matrix over std::threads, each taking a
contiguous chunk of observation rows, chunk = ceil(N / threads)
(matfill.hpp:206-221); entries are independent, so results do not depend on
the thread count.  Here the same chunking runs one rank per GPU:

1. every rank computes the pair-distance range of its own rows (K1),
2. ONE 16-byte all-reduce (MIN of {r_min, -r_max}) makes it global,
3. every rank builds the identical table from the global range (the device
   build is deterministic) and fills its rows -- no data-path collective,
4. optionally the row blocks are gathered to one rank (point-to-point sends
   into the destination's row slices; NVLink under NCCL), reported apart
   from the fill.

Works with any torch.distributed backend: NCCL on GPUs (tensors on the
rank's device), gloo on CPU (the tests).
"""
from __future__ import annotations


def rows_of(rank: int, world: int, N: int) -> tuple[int, int]:
    """Contiguous row block [begin, end) of `rank` (matfill.hpp:211-215)."""
    chunk = (N + world - 1) // world
    b = min(N, rank * chunk)
    return b, min(N, b + chunk)


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


def shard_summary(world: int, N: int) -> list[tuple[int, int]]:
    """All row blocks, rank order (for reports)."""
    return [rows_of(r, world, N) for r in range(world)]


def evals_of_rows(rows: int, N: int, m: int, n: int) -> int:
    """actual_calls of a row block: 3 m n rows (N - 1) (matfill.hpp:200)."""
    return 3 * m * n * rows * (N - 1) if N > 0 else 0


__all__ = ["rows_of", "global_distance_range", "gather_rows", "shard_summary", "evals_of_rows"]
