#!/usr/bin/env python3
"""Generate tests/golden/golden.npz from the REFERENCE itself.

Runs in the build container only (needs oracle/_ref/libgkref.so, compiled in
place from /root/reference by oracle/Makefile).  The fixtures pin the C
restatement (oracle/gk_oracle.c) in tests/test_golden.py on machines where the
reference tree is absent.  Re-run after changing any fixture definition:

    make -C oracle all && python tests/golden/make_golden.py
"""
import math
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.dirname(os.path.dirname(HERE)))

from oracle.pyoracle import (DIRECT, EXP, GREEN, TABLE, Oracle, Ref,  # noqa: E402
                             SamplingConfig, splitmix64_uniform)

# (name, SamplingConfig kwargs, medium (lambda0, eps_r, mu_r))
PLANS = [
    ("default", dict(), (1.0, 1.0, 1.0)),
    ("refine_off", dict(refine=False), (1.0, 1.0, 1.0)),
    ("c1_s1e3", dict(r_min=1e-3, r_max=2.0), (0.5, 1.0, 1.0)),
    ("c2_s1e3", dict(r_min=0.0118, r_max=1.9997), (1.0, 1.0, 1.0)),
    ("dielectric", dict(r_min=1e-3, r_max=1.3, samples_per_wavelength=700,
                        refine_interval_divisor=3, refine_halfwidth_in_t=2.5,
                        dedup_fraction=0.7), (0.8, 2.3, 1.7)),
    ("overlap_small_S", dict(samples_per_wavelength=20, refine_halfwidth_in_t=3.0),
     (1.0, 1.0, 1.0)),
]


def main():
    ref = Ref()
    out = {}
    for name, kw, med in PLANS:
        p = ref.build_plan(SamplingConfig(**kw), *med)
        b, dr, inv = ref.build_hash(p.abscissae, p.zeros)
        out[f"plan/{name}/abscissae"] = p.abscissae
        out[f"plan/{name}/zeros"] = p.zeros
        out[f"plan/{name}/t_dr"] = np.array([p.t, p.dr_min, inv])
        out[f"plan/{name}/buckets"] = b
    # evaluator on the reference configuration (test_evaluator.cpp:13-15)
    p = ref.build_plan(SamplingConfig(), 1.0, 1.0, 1.0)
    k = ref.wavenumber(1.0, 1.0, 1.0)
    ev = ref.evaluator(p, k)
    e, g = ev.tables()
    out["eval/exp_table"] = e
    out["eval/green_table"] = g
    r = splitmix64_uniform(4242, 4096, p.abscissae[0] / 10.0, p.abscissae[-1])
    out["eval/radii"] = r
    out["eval/exp"] = ev.eval_batch(EXP, r)
    out["eval/green"] = ev.eval_batch(GREEN, r)
    out["eval/fallbacks"] = np.array([ev.fallbacks], np.uint64)
    w = splitmix64_uniform(5, 4096, -1.0, 1.0)
    rr = splitmix64_uniform(6, 72, p.abscissae[0], p.abscissae[-1])
    out["acc/radii"], out["acc/weights"] = rr, w[:72]
    out["acc/value"] = np.array([ev.accumulate_green(rr, w[:72])])
    # fills: icosphere L0 (N=20) and jittered L1 (N=80)
    o = Oracle()
    v0, t0 = ref.sphere_mesh(0.5, 0)
    v1, t1 = ref.sphere_mesh(1.0, 1)
    v1 = o.jitter(v1, 1901, 1e-3)  # jitter is a workload generator (not in the reference)
    out["mesh/l1j/vertices"], out["mesh/l1j/triangles"] = v1, t1
    out["fill/l0_direct"], rep = ref.fill_matrix(v0, t0, 4, 3, DIRECT, 2 * math.pi)
    out["fill/l0_direct_calls"] = np.array([rep.actual_calls, rep.predicted_calls], np.uint64)
    hi = ref.max_vertex_distance(v0) * 1.01
    pt = ref.build_plan(SamplingConfig(r_min=1e-4, r_max=hi, samples_per_wavelength=10000))
    evt = ref.evaluator(pt, 2 * math.pi)
    out["fill/l0_table"], rep = ref.fill_matrix(v0, t0, 4, 3, TABLE, 2 * math.pi, ev=evt)
    out["fill/l0_table_plan"] = pt.abscissae
    out["fill/l1j_direct_m6n4"], _ = ref.fill_matrix(v1, t1, 6, 4, DIRECT, 2 * math.pi)
    out["fill/l1j_green_exp_m3n2"], _ = ref.fill_matrix(v1, t1, 3, 2, DIRECT, 2 * math.pi,
                                                        kind=EXP)
    # quadrature rules
    for m in (1, 3, 4, 6, 7):
        out[f"quad/tri{m}"] = ref.triangle_rule(m)
    for n in range(1, 8):
        out[f"quad/gl{n}"] = ref.gauss_legendre_unit(n)
    np.savez_compressed(os.path.join(HERE, "golden.npz"), **out)
    print(f"wrote {len(out)} arrays to {os.path.join(HERE, 'golden.npz')}")


if __name__ == "__main__":
    main()
