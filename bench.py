#!/usr/bin/env python3
"""Benchmark of the B200 MoM triangle-pair Green-function fill (arXiv 1901.04162).

One step = one full fill of the configuration's N x N complex128 matrix Z
(sharded by observation-row blocks over the ranks): TABLE mode = K1 pair
distance range (+ 16-byte NCCL all-reduce across ranks) + K2 device table
build + K3 fill; DIRECT mode = K4 fill (the reference charges the table build
to the table side, matfill.hpp:289-292).  Inputs (mesh, quadrature points)
are resident in HBM; the output (e.g. 107 GB for C5) is far larger than L2,
so no flush is needed between steps.

Default workload: BASELINE.json configs[4] (C5, icosphere L6, N = 81920,
m = 6, n = 4, k = 2 pi / 0.15), the metric's "vs N at 1/2/4/8 B200" config.
Rank 0 prints one JSON line.

* ``--gpus N`` with N > 1 and no WORLD_SIZE in the environment re-launches
  itself through ``torch.distributed.run`` (one rank per GPU, 127.0.0.1);
  under torchrun, WORLD_SIZE must equal N.
* ``--impl reference`` times the reference's own CPU fill (oracle/_ref,
  compiled in place from /root/reference) on the host cores, through
  oracle/cpu_bench.py -- the reference only: this package is never imported
  in that arm.  The GPU arm's ``cpu_baseline`` runs the same module in a clean
  subprocess.
* ``--selftest gloo`` runs the N-rank orchestration (self-launch, row blocks,
  barriers, max-over-ranks timing, the JSON line) on CPU ranks over gloo,
  with the reference's CPU fill of each rank's rows as the stand-in work: a
  harness test, not a bench number (``impl`` says so).
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

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

FLOPS_PER_EVAL = 44  # the reference's table-mode op count (FMA = 2)

CONFIGS = {
    "c2": dict(name="C2 icosphere L3 N=1280 m=6 n=4 lambda=1", kind="sphere", level=3, m=6, n=4,
               lambda0=1.0),
    "c3": dict(name="C3 icosphere L5 N=20480 m=7 n=5 lambda=0.3", kind="sphere", level=5, m=7,
               n=5, lambda0=0.3),
    "c4": dict(name="C4 plate 1m 100x100 N=20000 m=6 n=4 eps_r=4-0.4j lambda0=1", kind="plate",
               cells=100, m=6, n=4, lambda0=1.0, eps_r=4.0, eps_r_im=-0.4),
    "c5": dict(name="C5 icosphere L6 N=81920 m=6 n=4 lambda=0.15", kind="sphere", level=6, m=6,
               n=4, lambda0=0.15),
}
SEED, JITTER = 1901, 1e-3


def env_int(name, default):
    try:
        return int(os.environ.get(name, default))
    except ValueError:
        return default


def make_mesh(gk, cfg):
    if cfg["kind"] == "sphere":
        return gk.jitter(gk.generate_sphere_mesh(1.0, cfg["level"]), SEED, JITTER)
    return gk.generate_plate_mesh(1.0, cfg["cells"])


def rows_of(rank, world, N):
    """contiguous row blocks, chunk = ceil(N / world) (matfill.hpp:211-215);
    the same partition as paper_1901_04162_b200.sharding.rows_of and gk_rows_of"""
    chunk = (N + world - 1) // world
    b = min(N, rank * chunk)
    return b, min(N, b + chunk)


# the headline mode on both arms: the faster of the reference's two kernels
# (AnalyticKernel / TableKernel at S) -- same definition in both lines
MODE_NOTE = "faster of direct and table"
L2_NOTE = ("no flush needed: a step writes Z (rows x N x 16 B; 107 GB for the full C5 fill) "
           "far beyond any cache; the quadrature points (<= 47 MB) are re-read ~N times per "
           "step, so their cache residency is the steady state")


def config_of(cfg, S):
    """the `config` object, identical in both arms' lines"""
    return {"workload": cfg["name"], "mode": MODE_NOTE, "samples_per_wavelength": S,
            "l2": L2_NOTE}


def self_launch(args):
    """--gpus N > 1 without torchrun: re-exec as N ranks of torch.distributed.run."""
    import socket
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    env = dict(os.environ)
    if args.selftest is None:
        # the driver counts the communicator's ranks from NCCL's own log
        env.setdefault("NCCL_DEBUG", "INFO")
        env.setdefault("NCCL_DEBUG_SUBSYS", "INIT")
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1",
           f"--nproc-per-node={args.gpus}", "--master-addr", "127.0.0.1",
           "--master-port", str(port), os.path.abspath(__file__), *sys.argv[1:]]
    sys.stdout.flush()
    os.execvpe(sys.executable, cmd, env)


class ClockSampler:
    """SM clocks + throttle reasons sampled (NVML, every 50 ms) during the timed region."""

    REASONS = {"hw_slowdown": 0x8, "hw_thermal_slowdown": 0x40, "sw_thermal_slowdown": 0x20,
               "sw_power_cap": 0x4, "hw_power_brake_slowdown": 0x80}

    def __init__(self, index: int):
        self.index = index
        self.samples, self.reasons, self.max_mhz = [], set(), None
        self.err = None

    def _run(self):
        import pynvml as nv
        while not self.stop.is_set():
            try:
                self.samples.append(nv.nvmlDeviceGetClockInfo(self.h, nv.NVML_CLOCK_SM))
                bits = nv.nvmlDeviceGetCurrentClocksEventReasons(self.h)
                for nm, b in self.REASONS.items():
                    if bits & b:
                        self.reasons.add(nm)
            except Exception as exc:  # keep sampling
                self.err = repr(exc)
            self.stop.wait(0.05)

    def __enter__(self):
        import threading
        self.stop = threading.Event()
        try:
            import pynvml as nv
            nv.nvmlInit()
            vis = os.environ.get("CUDA_VISIBLE_DEVICES")
            idx = int(vis.split(",")[self.index]) if vis else self.index
            self.h = nv.nvmlDeviceGetHandleByIndex(idx)
            self.max_mhz = nv.nvmlDeviceGetMaxClockInfo(self.h, nv.NVML_CLOCK_SM)
            self.th = threading.Thread(target=self._run, daemon=True)
            self.th.start()
        except Exception as exc:
            self.err = repr(exc)
            self.th = None
        return self

    def __exit__(self, *exc):
        self.stop.set()
        if self.th:
            self.th.join(timeout=2)

    def summary(self):
        out = {"sm_mhz": statistics.median(self.samples) if self.samples else None,
               "sm_max_mhz": self.max_mhz, "samples": len(self.samples),
               "reasons": sorted(self.reasons)}
        if self.err and not self.samples:
            out["error"] = self.err
        return out


def cpu_threads():
    try:
        return len(os.sched_getaffinity(0))
    except AttributeError:
        return os.cpu_count() or 1


def cpu_baseline_subprocess(cfg, S, seconds, seconds_1):
    """The reference's CPU fill timed in a CLEAN subprocess (no torch, no CUDA
    context, no libgk.so): the same oracle/cpu_bench.py the reference arm runs,
    so the two CPU numbers measure the same code on the same workload."""
    import subprocess
    cmd = [sys.executable, "-m", "oracle.cpu_bench", "--level", str(cfg["level"]),
           "--m", str(cfg["m"]), "--n", str(cfg["n"]), "--lambda0", str(cfg["lambda0"]),
           "--S", str(S), "--seconds", str(seconds), "--seconds-1", str(seconds_1)]
    env = {k: v for k, v in os.environ.items() if not k.startswith(("CUDA_", "NCCL_"))}
    env["CUDA_VISIBLE_DEVICES"] = ""
    r = subprocess.run(cmd, capture_output=True, text=True, cwd=ROOT, env=env, timeout=900)
    if r.returncode != 0:
        raise RuntimeError(r.stderr.strip().splitlines()[-1] if r.stderr.strip() else "failed")
    return json.loads([ln for ln in r.stdout.splitlines() if ln.startswith("{")][-1])


def cpu_summary(res, S):
    """cpu_baseline from an oracle/cpu_bench result: the faster mode at nproc
    threads, both modes and the single-thread rates alongside."""
    modes = res["modes"]
    best = max(modes, key=lambda m: modes[m]["evals_per_s"])
    b = modes[best]
    kern = {"direct": "AnalyticKernel", "table": "TableKernel"}
    per = {}
    for m, e in modes.items():
        one = e.get("single_thread")
        per[m] = {"evals_per_s": e["evals_per_s"], "rows": e["rows"], "wall_s": e["wall_s"],
                  "threads": e["threads"],
                  "single_thread_evals_per_s": one["evals_per_s"] if one else None,
                  "single_thread_rows": one["rows"] if one else None}
        if m == "table":
            per[m].update(S=e["S"], table_build_ms=e["table_build_ms"],
                          table_nodes=e["table_nodes"])
    lo, hi = res.get("table_range", (None, None))
    return {"value": b["evals_per_s"], "unit": "evals/s", "cores": res["cores"],
            "kind": "reference", "mode": best, "modes": per,
            "single_thread": {"value": modes[best]["single_thread"]["evals_per_s"]
                              if modes[best].get("single_thread") else None,
                              "cores": 1, "mode": best},
            "sample": f"{b['rows']} of {res['N']} rows x all columns per sample through the "
                      f"reference's {kern[best]}::accumulate (the faster of its two modes; "
                      f"TableKernel at S={S} over [1e-4 lambda0, 1.01 max_vertex_distance]"
                      f"{f' = [{lo:.3g}, {hi:.5g}] m' if lo else ''}), {res['cores']} threads, "
                      f"extrapolated linearly to the {res['total_evals_per_fill']:.3e}-evaluation "
                      f"fill; single-thread rates alongside"}


def repo_libs_loaded():
    """this process's mapped shared objects under the repo (/proc/self/maps)"""
    out = set()
    try:
        with open("/proc/self/maps") as f:
            for ln in f:
                path = ln.split()[-1] if len(ln.split()) >= 6 else ""
                if path.startswith(ROOT) and ".so" in path:
                    out.add(os.path.relpath(path, ROOT))
    except OSError:
        pass
    return sorted(out)


def run_reference_arm(args, cfg, rank, world):
    """--impl reference: the reference's own CPU fill on this host's cores.

    Imports nothing of this package (only oracle/cpu_bench -> oracle/_ref/
    libgkref.so, the reference compiled in place).  Each step is a bounded
    row sample of the configured fill; ms_per_step is that
    sample's wall time, value its evaluations / s."""
    if rank != 0:
        return
    if cfg["kind"] != "sphere" or cfg.get("eps_r_im"):
        print(json.dumps({"impl": "reference", "unavailable":
                          "the reference is real-k only (kernel.hpp:23-24); C4 has no reference "
                          "path"}), flush=True)
        return
    from oracle.cpu_bench import Workload, cpu_threads, kernel_name
    wl = Workload(cfg["level"], cfg["m"], cfg["n"], cfg["lambda0"])
    threads = cpu_threads()
    modes = ["direct", "table"] if args.mode == "auto" else [args.mode]
    # every step a bounded sample: the whole K + W run stays within ~2-3 minutes
    per_step_s = min(args.cpu_seconds, max(1.0, 150.0 / (args.steps + args.warmup)))
    rows = {m: wl.rows_for(per_step_s, threads) for m in modes}
    warm = {m: [] for m in modes}
    for _ in range(args.warmup):      # warm-up samples of both modes pick the faster
        for m in modes:
            warm[m].append(wl.sample(m, rows[m], threads, args.S)["evals_per_s"])
    mode = max(modes, key=lambda m: statistics.median(warm[m]) if warm[m] else 0.0)
    timed = [wl.sample(mode, rows[mode], threads, args.S) for _ in range(args.steps)]
    evals = sum(t["evals"] for t in timed)
    wall = sum(t["wall_s"] for t in timed)
    v = evals / wall
    ms = wall / len(timed) * 1e3
    # single thread (threads = 1 and threads = nproc), once per mode
    single = {m: wl.sample(m, wl.rows_for(min(6.0, args.cpu_seconds) / len(modes), 1), 1, args.S)
              for m in modes} if args.cpu_single else {}
    per_mode = {m: {"evals_per_s": statistics.median(warm[m]) if warm[m] else None,
                    "rows": rows[m], "threads": threads,
                    "single_thread_evals_per_s": single[m]["evals_per_s"] if m in single else None,
                    "single_thread_rows": single[m]["rows"] if m in single else None}
                for m in modes}
    per_mode[mode]["evals_per_s"] = v
    if "table" in modes:
        ev, build_s, nodes = wl.evaluator(args.S)
        per_mode["table"].update(table_build_ms=build_s * 1e3, table_nodes=nodes)
    lo, hi = wl.table_range()
    line = {
        "impl": "reference", "metric": "green_fn_evals_per_s", "value": v, "unit": "evals/s",
        "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": ms, "higher_is_better": True, "scaling": "strong",
        "vs_baseline": None, "dtype": "f64",
        "data": "synthetic: the reference's generate_sphere_mesh + seeded jitter "
                "(splitmix64 seed 1901, 1e-3 m)",
        "config": config_of(cfg, args.S),
        "mode_used": mode,
        "parallelism": f"{threads} host threads (std::thread row chunks, matfill.hpp:206-221)",
        "step_definition": f"one bounded sample: {rows[mode]} of {wl.N} rows x all columns "
                           f"through the reference's {kernel_name(mode)}::accumulate "
                           f"(ms_per_step is the sample's wall time)",
        "full_fill_s_extrapolated": wl.total / v,
        "modes": per_mode,
        "cpu_baseline": {"value": v, "unit": "evals/s", "cores": threads, "kind": "reference",
                         "mode": mode,
                         "single_thread": {"value": single[mode]["evals_per_s"]
                                           if mode in single else None, "cores": 1},
                         "sample": f"{rows[mode]} rows x all {wl.N} columns per step through the "
                                   f"reference's {kernel_name(mode)}::accumulate (the faster of "
                                   f"its modes {sorted(modes)}; TableKernel at S={args.S} over "
                                   f"[{lo:.3g}, {hi:.5g}] m), extrapolated to the full "
                                   f"{wl.total:.3e}-eval fill"},
        "e2e": {"value": v, "unit": "evals/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
        "repo_libs_loaded": repo_libs_loaded(),
    }
    print(json.dumps(line), flush=True)


def run_selftest(args, cfg, rank, world):
    """--selftest gloo: the N-rank harness on CPU ranks (no GPU).  Each rank's
    step is the reference's CPU fill of a few rows of ITS row block; the step
    time is bracketed by barriers and reduced with MAX over ranks, exactly
    like the GPU arm.  Not a bench number."""
    import torch
    import torch.distributed as dist
    dist.init_process_group("gloo")
    assert dist.get_world_size() == world
    from oracle.cpu_bench import Workload
    wl = Workload(cfg["level"], cfg["m"], cfg["n"], cfg["lambda0"])
    rb, re = rows_of(rank, world, wl.N)
    import numpy as np
    rows = np.arange(rb, min(re, rb + 1 + rank), dtype=np.uint64)  # uneven work per rank

    def step():
        if rows.size:
            wl.ref.fill_sampled_rows(wl.verts, wl.tris, wl.m, wl.n, 0, wl.k, rows, threads=1)

    for _ in range(args.warmup):
        step()
    dist.barrier()
    t0 = time.perf_counter()
    for _ in range(args.steps):
        step()
    ms = (time.perf_counter() - t0) * 1e3 / args.steps
    dist.barrier()
    mine = torch.tensor([ms], dtype=torch.float64)
    allt = [torch.zeros(1, dtype=torch.float64) for _ in range(world)]
    dist.all_gather(allt, mine)
    mx = mine.clone()
    dist.all_reduce(mx, op=dist.ReduceOp.MAX)
    evals = torch.tensor([3.0 * wl.m * wl.n * rows.size * (wl.N - 1)], dtype=torch.float64)
    dist.all_reduce(evals)
    if rank == 0:
        print(json.dumps({
            "impl": f"selftest-{args.selftest}", "metric": "green_fn_evals_per_s",
            "value": float(evals[0]) / (float(mx[0]) * 1e-3), "unit": "evals/s",
            "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
            "ms_per_step": float(mx[0]), "per_rank_ms": [float(t[0]) for t in allt],
            "row_blocks": [list(rows_of(r, world, wl.N)) for r in range(world)],
            "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "f64",
            "data": "synthetic", "config": config_of(cfg, args.S),
            "note": "harness self-test on CPU ranks (gloo): not a bench value"}), flush=True)
    dist.destroy_process_group()


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="gk", choices=["gk", "reference"])
    ap.add_argument("--config", default="c5", choices=sorted(CONFIGS))
    ap.add_argument("--mode", default="auto", choices=["auto", "direct", "table"])
    ap.add_argument("--S", type=int, default=10000, help="samples per wavelength (table)")
    ap.add_argument("--both-modes", type=int, default=1, help="also time the other mode")
    ap.add_argument("--cpu-baseline", type=int, default=1)
    ap.add_argument("--cpu-seconds", type=float, default=10.0,
                    help="CPU wall budget per sample at nproc threads")
    ap.add_argument("--cpu-single", type=int, default=1,
                    help="also time the reference at threads = 1")
    ap.add_argument("--e2e", type=int, default=1)
    ap.add_argument("--vs-n", type=int, default=1, help="also time C2/C3 fills (rank 0, N=1)")
    ap.add_argument("--c1", type=int, default=1, help="also time standalone eval_batch (C1)")
    ap.add_argument("--gather", type=int, default=1,
                    help="N > 1: also time the gather of Z to rank 0 (reported apart)")
    ap.add_argument("--pertri", type=int, default=1,
                    help="also time the direct fill without shared edges (shared_edges = 0)")
    ap.add_argument("--S-alt", type=int, default=1000,
                    help="also time the table mode at this S (0 = off)")
    ap.add_argument("--selftest", default=None, choices=["gloo"],
                    help="CPU-only harness test of the N-rank orchestration")
    args = ap.parse_args()
    if args.warmup < 3:
        args.warmup = 3  # timing rule: >= 3 warm-up steps

    cfg = CONFIGS[args.config]
    if args.impl == "reference":
        # rank 0 alone runs the host-CPU reference; other torchrun ranks exit 0
        run_reference_arm(args, cfg, env_int("RANK", 0), env_int("WORLD_SIZE", args.gpus))
        return
    if "WORLD_SIZE" not in os.environ and args.gpus > 1:
        self_launch(args)  # does not return
    world = env_int("WORLD_SIZE", 1)
    if world != args.gpus:
        sys.stderr.write(f"bench.py: --gpus {args.gpus} but WORLD_SIZE={world}\n")
        sys.exit(2)
    rank = env_int("RANK", 0)
    local = env_int("LOCAL_RANK", 0)
    if args.selftest:
        run_selftest(args, cfg, rank, world)
        return
    run_gpu_arm(args, cfg, rank, world, local)


def run_gpu_arm(args, cfg, rank, world, local):
    import torch
    import torch.distributed as dist
    torch.cuda.set_device(local)
    comm = None
    if world > 1:
        os.environ.setdefault("NCCL_DEBUG", "INFO")
        os.environ.setdefault("NCCL_DEBUG_SUBSYS", "INIT")
        dist.init_process_group("nccl", device_id=torch.device(f"cuda:{local}"))
        comm = {"backend": dist.get_backend(), "world_size": dist.get_world_size()}
        sys.stderr.write(f"bench.py rank {rank}: torch.distributed {comm['backend']} "
                         f"nranks={comm['world_size']}\n")
    import paper_1901_04162_b200 as gk
    from paper_1901_04162_b200 import sharding
    from paper_1901_04162_b200._lib import lib as _gk_lib
    gk_lib = _gk_lib()

    ctx = gk.Context.get(local)
    mesh = make_mesh(gk, cfg)
    N = mesh.triangle_count()
    m, n = cfg["m"], cfg["n"]
    spec = gk.QuadratureSpec(m, n)
    medium = gk.Medium(lambda0=cfg["lambda0"], eps_r=cfg.get("eps_r", 1.0),
                       eps_r_im=cfg.get("eps_r_im", 0.0))
    k = gk.wavenumber(medium)
    rb, re = rows_of(rank, world, N)
    assert (rb, re) == sharding.rows_of(rank, world, N)
    rows = re - rb
    dmesh = gk.DeviceMesh(mesh, spec, ctx)
    Z = torch.empty((max(rows, 1), N), dtype=torch.complex128, device=f"cuda:{local}")
    total_evals = 3 * m * n * N * (N - 1)
    # the reference-order kernels (no shared edges): A/B only
    per_tri = gk.FillOptions(shared_edges=0)
    # N > 1: libgk's own NCCL communicator (C++, csrc/comm.cu); every step is
    # gk_fill_sharded: K1 on the rank's rows + the 16-byte device all-reduce +
    # table build (TABLE) + the fill of its rows
    gkcomm = None
    if world > 1:
        gkcomm = sharding.Comm(ctx)
        comm["gk_comm_nranks"] = gkcomm.info()[0]

    def global_range():
        if gkcomm is not None:
            return sharding.distance_range_global(gkcomm, dmesh)
        return dmesh.distance_range(rb, re)

    def table_for(mode):
        if not mode.startswith("table"):
            return None
        S = args.S if mode == "table" else int(mode.split("_S")[1])
        lo, hi = global_range()
        return gk.DeviceTable(gk.SamplingConfig(r_min=lo, r_max=hi, samples_per_wavelength=S),
                              medium, ctx=ctx)

    fill_ev = []

    def sharded_step(mode, report):
        S = args.S if mode in ("table", "direct", "direct_pertri") else int(mode.split("_S")[1])
        cfg_s = gk.SamplingConfig(r_min=0.0, r_max=0.0, samples_per_wavelength=S)
        rep, _ = sharding.fill_rows_sharded(
            gkcomm, dmesh, gk.Mode.TABLE if mode.startswith("table") else gk.Mode.DIRECT, Z,
            cfg=cfg_s, medium=medium, options=per_tri if mode == "direct_pertri" else None,
            report=report)
        return rep

    def step(mode):
        e0 = torch.cuda.Event(enable_timing=True)
        e1 = torch.cuda.Event(enable_timing=True)
        if gkcomm is not None:
            e0.record()
            sharded_step(mode, False)
            e1.record()
            fill_ev.append((e0, e1))
            return None
        table = table_for(mode)
        e0.record()
        if rows:
            gk.fill_rows(dmesh, gk.Mode.TABLE if table else gk.Mode.DIRECT, table=table, k=k,
                         row_begin=rb, row_end=re, out=Z, report=False,
                         options=per_tri if mode == "direct_pertri" else None)
        e1.record()
        fill_ev.append((e0, e1))
        return table

    launches = {}

    def timed(mode, steps, warmup):
        for _ in range(warmup):
            step(mode)
        torch.cuda.synchronize()
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize()
        fill_ev.clear()
        l0 = gk_lib.gk_launch_count()
        s0 = torch.cuda.Event(enable_timing=True)
        s1 = torch.cuda.Event(enable_timing=True)
        s0.record()
        for _ in range(steps):
            step(mode)
        s1.record()
        torch.cuda.synchronize()
        launches[mode] = gk_lib.gk_launch_count() - l0
        if world > 1:
            dist.barrier()
        ms = s0.elapsed_time(s1) / steps
        fill_ms = sum(a.elapsed_time(b) for a, b in fill_ev) / len(fill_ev)
        if world > 1:
            t = torch.tensor([ms, fill_ms], dtype=torch.float64, device=f"cuda:{local}")
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
            ms, fill_ms = float(t[0]), float(t[1])
        return ms, fill_ms

    def performed_evals(mode):
        """(evaluations the kernel performs per step, the fill kernel's name)"""
        if gkcomm is not None:
            rep = sharded_step(mode, True)
            return rep.evaluations, rep.path_name
        if not rows:
            return 0, "none"
        table = table_for(mode)
        _, rep = gk.fill_rows(dmesh, gk.Mode.TABLE if table else gk.Mode.DIRECT, table=table,
                              k=k, row_begin=rb, row_end=re, out=Z,
                              options=per_tri if mode == "direct_pertri" else None)
        return rep.evaluations, rep.path_name

    # roofline denominator: FP64 DFMA peak measured on this device now
    p64 = ctx.fp64_peak_tflops()
    modes = ["direct", "table"] if args.mode == "auto" or args.both_modes else [args.mode]
    if args.mode != "auto":
        modes = [args.mode] + ([x for x in ("direct", "table") if x != args.mode]
                               if args.both_modes else [])
    if args.S_alt and args.S_alt != args.S and "table" in modes:
        modes.append(f"table_S{args.S_alt}")
    if args.pertri and "direct" in modes:
        modes.insert(modes.index("direct") + 1, "direct_pertri")
    results = {}
    clocks = None
    for i, mode in enumerate(modes):
        steps = args.steps if i == 0 else max(1, min(args.steps, 3))
        if i == 0:
            with ClockSampler(local) as cs:
                ms, fill_ms = timed(mode, steps, args.warmup)
            clocks = cs.summary()
        else:
            ms, fill_ms = timed(mode, steps, 1)
        # evaluations the kernel performs per launch (fewer than the
        # reference's calls on the shared-edge paths): one synchronous fill
        # outside the timed region reports them
        performed, path = performed_evals(mode)
        evals_all = performed
        if world > 1:
            t = torch.tensor([performed], dtype=torch.float64, device=f"cuda:{local}")
            dist.all_reduce(t)
            evals_all = float(t[0])
        results[mode] = {"kernel": path, "ms_per_step": ms, "fill_kernel_ms": fill_ms,
                         "evals_per_s": total_evals / (ms * 1e-3),
                         "evaluations_per_step": evals_all,
                         "evaluations_performed_per_s": evals_all / (ms * 1e-3),
                         "kernel_tflops": performed * FLOPS_PER_EVAL / (fill_ms * 1e-3) / 1e12}
    # the timed fills ran asynchronously: surface any fallback / range / r = 0
    # error now (outside the timed region), like a synchronous fill would
    ctx.fill_check()

    # the headline mode: the faster of direct and the table at the configured S
    chosen = args.mode if args.mode != "auto" else min(("direct", "table"),
                                                       key=lambda x: results[x]["ms_per_step"])
    main_res = results[chosen]

    # e2e through the host-buffer C-ABI entry point (gk_fill_matrix_host), rank-local rows
    e2e = None
    if args.e2e:
        e2e = run_e2e(gk, ctx, cfg, mesh, spec, medium, chosen, args, total_evals, rank, world,
                      rb, re, dist if world > 1 else None, gkcomm)

    vs_n = None
    if args.vs_n and rank == 0 and world == 1 and args.config == "c5":
        vs_n = run_vs_n(gk, ctx, chosen, args)

    gather = None
    if world > 1 and args.gather:
        gather = run_gather(sharding, gkcomm, Z, N, rows, local, dist)
        if "ms" in gather:
            gather["fused"] = run_fused_gather(gk, sharding, dmesh, chosen, medium, k, args, N,
                                               rows, local, dist, global_range)

    c1 = None
    if args.c1 and rank == 0 and world == 1:
        c1 = run_c1(gk, ctx)

    # the reference's CPU fill beside it (rank 0, N = 1): a clean subprocess
    # running oracle/cpu_bench.py -- the code the reference arm runs
    cpu = None
    if args.cpu_baseline and rank == 0 and world == 1:
        if cfg["kind"] != "sphere" or cfg.get("eps_r_im"):
            cpu = {"value": None, "unit": "evals/s", "cores": cpu_threads(), "kind": "reference",
                   "sample": "unavailable: the reference is real-k only (kernel.hpp:23-24)"}
        else:
            try:
                cpu = cpu_summary(cpu_baseline_subprocess(
                    cfg, args.S, args.cpu_seconds, min(6.0, args.cpu_seconds) if args.cpu_single
                    else 0.0), args.S)
            except Exception as exc:  # report, never fake
                cpu = {"value": None, "unit": "evals/s", "cores": cpu_threads(),
                       "kind": "reference", "sample": f"unavailable: {exc}"}

    traffic = None
    tpath = os.path.join(ROOT, "profiles", "traffic.json")
    if os.path.exists(tpath):
        try:
            traffic = json.load(open(tpath)).get(f"{args.config}:{chosen}")
        except (OSError, ValueError):
            traffic = None

    fill_bytes = rows * N * 16
    line = {
        "metric": "green_fn_evals_per_s",
        "value": main_res["evals_per_s"],
        "unit": "evals/s",
        "n_gpus": world,
        "steps": args.steps,
        "warmup": args.warmup,
        "ms_per_step": main_res["ms_per_step"],
        "higher_is_better": True,
        "scaling": "strong",
        "vs_baseline": None,
        "dtype": "f64",
        "data": "synthetic: seeded jittered icosphere (splitmix64 seed 1901, 1e-3 m)",
        "config": config_of(cfg, args.S),
        "mode_used": chosen,
        "parallelism": f"row-block x{world}",
        "comm": comm,
        "fill_time_s": main_res["ms_per_step"] * 1e-3,
        "value_definition": "the reference's calls per Z fill (FillReport.actual_calls = "
                            "3 m n N (N-1), matfill.hpp:200) / fill time, i.e. Z-fill time "
                            "expressed as Green-function evaluations of the reference's "
                            "algorithm; the direct kernel evaluates each shared mesh edge "
                            "once for both triangles, performing evaluations_per_step of them "
                            "(roofline.achieved counts only those)",
        "evaluations_per_step": main_res["evaluations_per_step"],
        "evaluations_performed_per_s": main_res["evaluations_performed_per_s"],
        "roofline": {"bound": "fp64", "achieved": main_res["kernel_tflops"], "peak": p64,
                     "peak_nominal": 148 * 64 * 2 * 1.965e9 / 1e12,
                     "unit": "TFLOP/s", "frac": main_res["kernel_tflops"] / p64,
                     "traffic": traffic,
                     "note": f"{FLOPS_PER_EVAL} algorithmic FP64 flops/eval (SURVEY 8d, FMA=2) x "
                             f"evaluations performed per launch / fill-kernel event time; peak = DFMA "
                             f"microbenchmark on this GPU (MEASURED_PEAKS.json has no FP64 entry)",
                     "hbm_write_gbs": fill_bytes / (main_res["fill_kernel_ms"] * 1e-3) / 1e9},
        "modes": results,
        "clocks": clocks,
        "gpu_launches": launches[chosen],
        "cpu_baseline": cpu,
        "e2e": e2e,
    }
    if vs_n:
        line["vs_N"] = vs_n
    if c1:
        line["c1_eval_batch"] = c1
    if gather:
        line["gather"] = gather
    if rank == 0:
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.destroy_process_group()


def run_e2e(gk, ctx, cfg, mesh, spec, medium, mode, args, total_evals, rank, world, rb, re,
            dist=None, gkcomm=None):
    """End to end through the C-ABI host-buffer entry points, at N ranks: each
    step every rank uploads the host mesh (H2D), generates its quadrature
    points, (TABLE) computes its range, all-reduces it and builds the table,
    fills its row block and copies every byte of it to pinned host memory
    (D2H).  At N = 1 a Z that fits host RAM (C2-C4) goes through
    gk_fill_matrix_host into a full host matrix; larger row blocks (C5: 107 GB
    / N) are streamed with gk_fill_rows_host into a reused 4 GiB pinned host
    window (the full matrix does not fit this host's RAM twice, nor the
    reference's).  Time = max over ranks."""
    import torch
    N = mesh.triangle_count()
    rows = re - rb
    nbytes = rows * N * 16
    full = world == 1 and nbytes <= (16 << 30)
    rows_win = max(1, min(rows, (4 << 30) // (N * 16)))
    try:
        zh = torch.empty((rows_win if not full else N, N), dtype=torch.complex128, pin_memory=True)
    except RuntimeError as exc:
        return {"value": None, "unit": "evals/s", "h2d_bytes_per_step": 0,
                "d2h_bytes_per_step": N * N * 16, "note": f"pinned host buffer unavailable: {exc}"}
    z = zh.numpy()
    m = gk.Mode.TABLE if mode == "table" else gk.Mode.DIRECT
    k = gk.wavenumber(medium)
    # the step's inputs (the mesh) live in pinned host memory, copied in every step
    pv = torch.from_numpy(mesh.vertices).pin_memory()
    pt = torch.from_numpy(mesh.triangles.view(np.int32)).pin_memory()
    mesh = gk.TriangleMesh(pv.numpy(), pt.numpy().view(np.uint32))
    assert mesh.vertices.ctypes.data == pv.data_ptr()   # no copy: the pinned buffers

    def step():
        if full:
            cfgs = gk.SamplingConfig(r_min=0.0, r_max=0.0, samples_per_wavelength=args.S)
            gk.fill_matrix(mesh, spec, m, medium, cfgs, ctx=ctx, out=z)
            return
        dm = gk.DeviceMesh(mesh, spec, ctx)
        t = None
        if m == gk.Mode.TABLE:
            if gkcomm is not None:   # K1 on this rank's rows + the NCCL all-reduce (C++)
                from paper_1901_04162_b200.sharding import distance_range_global
                lo, hi = distance_range_global(gkcomm, dm)
            else:
                lo, hi = dm.distance_range(rb, re)
            t = gk.DeviceTable(gk.SamplingConfig(r_min=lo, r_max=hi,
                                                 samples_per_wavelength=args.S), medium, ctx=ctx)
        for b in range(rb, re, rows_win):
            gk.fill_rows_host(dm, m, z, table=t, k=k, row_begin=b, row_end=min(re, b + rows_win))

    step()  # warm-up
    steps = max(1, min(args.steps, 3))
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    t0 = time.perf_counter()
    for _ in range(steps):
        step()
    dt = (time.perf_counter() - t0) / steps
    if world > 1:
        tt = torch.tensor([dt], dtype=torch.float64, device=f"cuda:{ctx.device}")
        dist.all_reduce(tt, op=dist.ReduceOp.MAX)
        dt = float(tt[0])
    h2d = (mesh.vertices.nbytes + mesh.triangles.nbytes) * world
    return {"value": total_evals / dt, "unit": "evals/s", "h2d_bytes_per_step": int(h2d),
            "d2h_bytes_per_step": int(N * N * 16), "ms_per_step": dt * 1e3,
            "api": ("gk_fill_matrix_host -> full pinned host Z" if full else
                    f"per rank: gk_mesh_create + gk_fill_rows_host x{(rows + rows_win - 1) // rows_win}"
                    f" -> {rows_win}-row pinned host window"),
            "timing": "host wall clock per step, max over ranks"}


def run_gather(sharding, gkcomm, Z, N, rows, local, dist):
    """Optional gather of all row blocks of Z to rank 0 (gk_gather_rows:
    grouped ncclSend / ncclRecv over NVLink from C++), timed apart from the
    fill.  Skipped when the full matrix does not fit next
    to rank 0's own block."""
    import torch
    need = N * N * 16
    ok = torch.tensor([1.0 if torch.cuda.mem_get_info(local)[0] > need + (4 << 30) else 0.0],
                      device=f"cuda:{local}")
    dist.all_reduce(ok, op=dist.ReduceOp.MIN)
    if ok.item() == 0:
        return {"skipped": f"full Z ({need / 1e9:.1f} GB) does not fit rank 0's free memory"}
    out = torch.empty((N, N), dtype=torch.complex128, device=f"cuda:{local}") \
        if dist.get_rank() == 0 else None
    torch.cuda.synchronize()
    dist.barrier()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    sharding.gather_rows_nccl(gkcomm, Z, N, root=0, out=out)
    e1.record()
    torch.cuda.synchronize()
    t = torch.tensor([e0.elapsed_time(e1)], dtype=torch.float64, device=f"cuda:{local}")
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    ms = float(t[0])
    del out
    torch.cuda.empty_cache()   # the fused variant allocates the full matrix outside torch
    return {"ms": ms, "bytes": need, "gbs": need / (ms * 1e-3) / 1e9,
            "how": "row blocks sent to rank 0 after the fill (gk_gather_rows: grouped "
                   "ncclSend/ncclRecv in libgk, C++)"}


def run_fused_gather(gk, sharding, dmesh, mode, medium, k, args, N, rows, local, dist,
                     global_range):
    """Fill + gather fused: every rank's fill kernel stores its rows straight
    into rank 0's matrix through CUDA IPC peer memory (NVLink), no separate
    collective (sharding.fill_rows_gathered).  Device time, max over ranks."""
    import torch
    table = None
    if mode == "table":
        lo, hi = global_range()
        table = gk.DeviceTable(gk.SamplingConfig(r_min=lo, r_max=hi,
                                                 samples_per_wavelength=args.S), medium)
    m = gk.Mode.TABLE if table else gk.Mode.DIRECT
    try:
        torch.cuda.synchronize()
        dist.barrier()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        full, _ = sharding.fill_rows_gathered(dmesh, m, table=table, k=k)
        e1.record()
        torch.cuda.synchronize()
        del full
    except Exception as exc:  # report, never fake
        return {"unavailable": repr(exc)[:200]}
    t = torch.tensor([e0.elapsed_time(e1)], dtype=torch.float64, device=f"cuda:{local}")
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return {"ms": float(t[0]), "mode": mode,
            "how": "each rank's fill kernel writes its row block into rank 0's matrix via "
                   "CUDA IPC peer stores (fill + gather in one pass)"}


def hbm_peak_gbs():
    try:
        return float(json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))["hbm_gbs"]), \
            "MEASURED_PEAKS.json hbm_gbs (copy, burst)"
    except (OSError, ValueError, KeyError):
        return 6650.0, "fallback 6.65 TB/s (B200_PROFILING.md; MEASURED_PEAKS.json absent)"


def run_c1(gk, ctx, iters=1024, sets=8):
    """C1 (BASELINE configs[0]): standalone eval_batch of 2^20 seeded radii in
    [1e-3, 2] m, k = 4 pi, through gk_eval_batch_async, `iters` back-to-back
    launches rotating over `sets` radius/output buffers (192 MB > L2, so every
    launch streams from HBM).  Algorithmic bytes: 8 B read + 16 B written per
    radius; the table itself stays cache-resident."""
    import torch
    n = 1 << 20
    dev = f"cuda:{ctx.device}"
    rng = np.random.default_rng(1901)
    rs = [torch.as_tensor(rng.uniform(1e-3, 2.0, n), device=dev) for _ in range(sets)]
    outs = [torch.empty(n, dtype=torch.complex128, device=dev) for _ in range(sets)]
    med = gk.Medium(lambda0=0.5)
    k = gk.wavenumber(med)
    st = gk.EvalStatus(ctx)
    peak, peak_src = hbm_peak_gbs()
    res = {"n": n, "iters": iters, "bytes_per_eval": 24, "peak_gbs": peak, "peak": peak_src}
    variants = [("direct", None)] + [(f"table_S{S}", S) for S in (1000, 10000)]
    res["graph"] = "the same launches captured once in a CUDA graph and replayed"
    for name, S in variants:
        t = None
        if S:
            t = gk.DeviceTable(gk.SamplingConfig(r_min=1e-3, r_max=2.0, samples_per_wavelength=S),
                               med, ctx=ctx)
        for kind in (gk.KernelKind.PlainExp, gk.KernelKind.GreenOverR):
            def run():
                for i in range(iters):
                    gk.eval_batch_async(kind, rs[i % sets], outs[i % sets], st, table=t, k=k)
            for i in range(2 * sets):  # warm-up
                gk.eval_batch_async(kind, rs[i % sets], outs[i % sets], st, table=t, k=k)
            torch.cuda.synchronize()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            run()
            e1.record()
            torch.cuda.synchronize()
            us = e0.elapsed_time(e1) * 1e3 / iters
            # CUDA graph of the same launches (no per-launch host overhead)
            g = torch.cuda.CUDAGraph()
            side = torch.cuda.Stream()
            side.wait_stream(torch.cuda.current_stream())
            with torch.cuda.stream(side):
                with torch.cuda.graph(g, stream=side):
                    ctx.bind_stream()
                    run()
            ctx.bind_stream()
            g.replay()
            torch.cuda.synchronize()
            e0.record()
            g.replay()
            e1.record()
            torch.cuda.synchronize()
            ug = e0.elapsed_time(e1) * 1e3 / iters
            st.read()
            del g
            gbs, gbs_g = n * 24 / (us * 1e-6) / 1e9, n * 24 / (ug * 1e-6) / 1e9
            res[f"{name}:{'exp' if kind == gk.KernelKind.PlainExp else 'green'}"] = {
                "us_per_batch": us, "evals_per_s": n / (us * 1e-6), "gbs": gbs,
                "hbm_frac": gbs / peak, "graph_us_per_batch": ug,
                "graph_evals_per_s": n / (ug * 1e-6), "graph_hbm_frac": gbs_g / peak}
        st.reset()
    return res


def run_vs_n(gk, ctx, mode, args):
    """Z-fill time vs N on one GPU for the other sphere configs (informational)."""
    import torch
    out = {}
    for key in ("c2", "c3"):
        cfg = CONFIGS[key]
        mesh = make_mesh(gk, cfg)
        N = mesh.triangle_count()
        dm = gk.DeviceMesh(mesh, gk.QuadratureSpec(cfg["m"], cfg["n"]), ctx)
        med = gk.Medium(lambda0=cfg["lambda0"])
        k = gk.wavenumber(med)
        Z = torch.empty((N, N), dtype=torch.complex128, device=f"cuda:{ctx.device}")

        def once():
            t = None
            if mode == "table":
                lo, hi = dm.distance_range()
                t = gk.DeviceTable(gk.SamplingConfig(r_min=lo, r_max=hi,
                                                     samples_per_wavelength=args.S), med, ctx=ctx)
            gk.fill_rows(dm, gk.Mode.TABLE if t else gk.Mode.DIRECT, table=t, k=k, out=Z,
                         report=False)
        for _ in range(3):
            once()
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        reps = 20 if key == "c2" else 3
        e0.record()
        for _ in range(reps):
            once()
        e1.record()
        torch.cuda.synchronize()
        ms = e0.elapsed_time(e1) / reps
        ev = 3 * cfg["m"] * cfg["n"] * N * (N - 1)
        out[key] = {"N": N, "fill_ms": ms, "evals_per_s": ev / (ms * 1e-3)}
        del Z
    return out


if __name__ == "__main__":
    main()
