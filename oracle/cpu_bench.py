"""CPU baseline of the fill: the reference's own fill on this host's cores.

TEST / BENCH INFRASTRUCTURE ONLY (the checker and the CPU baseline, never the
product).  This module is the ONE implementation behind both CPU numbers
bench.py reports:

* ``bench.py --impl reference`` (the driver's reference arm) imports it
  directly, and
* the GPU arm's ``cpu_baseline`` leg runs it as a clean subprocess
  (``python -m oracle.cpu_bench``) -- no torch, no CUDA context, no libgk.so
  in that process -- so both arms measure the same code on the same workload.

Everything it loads is the reference compiled in place
(``oracle/_ref/libgkref.so``, built by ``oracle/Makefile`` from
``/root/reference/proj/include``):

* mesh: the reference's ``generate_sphere_mesh`` (mesh.hpp:154-202, via
  ``gr_sphere_mesh``) + the workload's seeded splitmix64 jitter restated in
  numpy below (bit-identical to ``gk_jitter`` / ``go_jitter``; the reference
  has no jitter);
* table range: the reference's own conventions -- r_max = 1.01 x
  ``max_vertex_distance`` (matfill.hpp:270, mesh.hpp:62-68), r_min = 1e-4 x
  lambda0 (gktab_main.cpp:62);
* fill: ``gr_fill_sampled_rows`` -- the reference's ``AnalyticKernel`` /
  ``TableKernel::accumulate`` (matfill.hpp:59-87) inside fill_rows' staging
  loop (matfill.hpp:185-199), rows split over std::threads in contiguous
  chunks like matfill.hpp:206-221.

The full C5 fill (4.8e11 evaluations, 2 x 107 GB of host RAM for the
reference's bench_compare) does not fit a bounded run, so each sample is a
deterministic row subset p = floor(s N / R) and the rate is
extrapolated linearly (every row costs N - 1 entries).
"""
from __future__ import annotations

import argparse
import json
import math
import os
import statistics
import sys
import time

import numpy as np

if __package__ in (None, ""):
    sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

from oracle.pyoracle import DIRECT, TABLE, Ref, SamplingConfig  # noqa: E402

SEED, JITTER = 1901, 1e-3
# the reference's measured per-thread rate on these boxes is ~15-20 ns per
# evaluation; used only to size a sample to a wall-time budget
NS_PER_EVAL_THREAD = 20e-9


def jitter(verts: np.ndarray, seed: int = SEED, amp: float = JITTER) -> np.ndarray:
    """splitmix64(seed) per coordinate in x, y, z order, U(-amp, amp) from the
    top 53 bits: the same arithmetic as go_jitter (gk_oracle.c) and gk_jitter
    (csrc/host.cpp), op by op (numpy rounds each operation; no contraction)."""
    v = np.ascontiguousarray(verts, np.float64).reshape(-1).copy()
    n = v.size
    ctr = (np.arange(1, n + 1, dtype=np.uint64) * np.uint64(0x9E3779B97F4A7C15)
           + np.uint64(seed))
    with np.errstate(over="ignore"):
        z = (ctr ^ (ctr >> np.uint64(30))) * np.uint64(0xBF58476D1CE4E5B9)
        z = (z ^ (z >> np.uint64(27))) * np.uint64(0x94D049BB133111EB)
        z = z ^ (z >> np.uint64(31))
    u = (z >> np.uint64(11)).astype(np.float64) * (2.0 ** -53)
    v += amp * (2.0 * u - 1.0)
    return v.reshape(verts.shape)


def cpu_threads() -> int:
    try:
        return len(os.sched_getaffinity(0))
    except AttributeError:
        return os.cpu_count() or 1


class Workload:
    """A sphere config (C2/C3/C5) built through the reference only."""

    def __init__(self, level: int, m: int, n: int, lambda0: float, ref: Ref | None = None):
        self.ref = ref or Ref()
        v, t = self.ref.sphere_mesh(1.0, level)
        self.verts, self.tris = jitter(v), t
        self.N = t.shape[0]
        self.m, self.n, self.lambda0 = m, n, lambda0
        self.k = self.ref.wavenumber(lambda0)
        self.per_row = 3 * m * n * (self.N - 1)
        self.total = self.per_row * self.N
        self._ev = {}

    def table_range(self) -> tuple[float, float]:
        """(r_min, r_max) by the reference's own conventions."""
        return 1e-4 * self.lambda0, 1.01 * self.ref.max_vertex_distance(self.verts)

    def evaluator(self, S: int):
        """build_plan + KernelEvaluator (timed: charged to the table side)."""
        if S not in self._ev:
            lo, hi = self.table_range()
            t0 = time.perf_counter()
            plan = self.ref.build_plan(SamplingConfig(r_min=lo, r_max=hi,
                                                      samples_per_wavelength=S), self.lambda0)
            ev = self.ref.evaluator(plan, self.k)
            self._ev[S] = (ev, time.perf_counter() - t0, plan.abscissae.size)
        return self._ev[S]

    def rows_for(self, seconds: float, threads: int) -> int:
        R = int(seconds * threads / (self.per_row * NS_PER_EVAL_THREAD))
        R = max(threads, (R // threads) * threads)
        return min(self.N, R)

    def sample(self, mode: str, rows: int, threads: int, S: int = 10000) -> dict:
        """One row-sampled reference fill; rate = evaluations / wall."""
        rws = np.array([(s * self.N) // rows for s in range(rows)], np.uint64)
        ev, build_s, nodes = (None, 0.0, 0)
        if mode == "table":
            ev, build_s, nodes = self.evaluator(S)
        _, calls, wall = self.ref.fill_sampled_rows(
            self.verts, self.tris, self.m, self.n, TABLE if ev is not None else DIRECT,
            self.k, rws, ev=ev, threads=threads)
        out = {"mode": mode, "threads": threads, "rows": rows, "evals": int(calls),
               "wall_s": wall, "evals_per_s": calls / wall}
        if mode == "table":
            out.update(S=S, table_build_ms=build_s * 1e3, table_nodes=int(nodes))
        return out


def kernel_name(mode: str) -> str:
    return "TableKernel" if mode == "table" else "AnalyticKernel"


def measure(wl: Workload, modes, S: int, seconds_nproc: float, seconds_1: float,
            repeats: int = 1) -> dict:
    """Both thread counts SURVEY 8d asks for (threads = nproc and 1), every
    mode; median of `repeats` samples at nproc."""
    nproc = cpu_threads()
    res = {"cores": nproc, "N": wl.N, "total_evals_per_fill": wl.total, "modes": {}}
    for mode in modes:
        rows = wl.rows_for(seconds_nproc / len(modes), nproc)
        runs = [wl.sample(mode, rows, nproc, S) for _ in range(max(1, repeats))]
        best = statistics.median(r["evals_per_s"] for r in runs)
        entry = dict(runs[0])
        entry["evals_per_s"] = best
        one = None
        if seconds_1 > 0:
            r1 = wl.rows_for(seconds_1 / len(modes), 1)
            one = wl.sample(mode, r1, 1, S)
        entry["single_thread"] = one
        res["modes"][mode] = entry
    return res


def main(argv=None) -> int:
    ap = argparse.ArgumentParser(description=__doc__.split("\n")[0])
    ap.add_argument("--level", type=int, required=True)
    ap.add_argument("--m", type=int, required=True)
    ap.add_argument("--n", type=int, required=True)
    ap.add_argument("--lambda0", type=float, required=True)
    ap.add_argument("--S", type=int, default=10000)
    ap.add_argument("--modes", default="direct,table")
    ap.add_argument("--seconds", type=float, default=10.0, help="wall budget at nproc threads")
    ap.add_argument("--seconds-1", type=float, default=6.0, help="wall budget at 1 thread")
    ap.add_argument("--repeats", type=int, default=1)
    a = ap.parse_args(argv)
    wl = Workload(a.level, a.m, a.n, a.lambda0)
    res = measure(wl, a.modes.split(","), a.S, a.seconds, a.seconds_1, a.repeats)
    res["table_range"] = list(wl.table_range())
    print(json.dumps(res), flush=True)
    return 0


if __name__ == "__main__":
    sys.exit(main())
