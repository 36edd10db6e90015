"""Generates tests/golden/*.json by running the REFERENCE ITSELF (oracle/_ref,
compiled from /root/reference/proj/src by oracle/Makefile) on seeded inputs.

TEST INFRASTRUCTURE ONLY. Inputs follow SURVEY.md §8(d): f from
std::mt19937(seed_f=1) + uniform_real_distribution(-1,1) over the finest interior
(row-major, x fastest), start vector zero or seed_x=2; b = f.

    python oracle/make_golden.py            # all fast fixtures (< 2 min)
    python oracle/make_golden.py c4         # the 8191^2 history (~5 min of CPU)
    python oracle/make_golden.py c2         # the 12 anisotropic Gauss-Seidel cases (~3 min)
    python oracle/make_golden.py c5         # one 16383^2 cycle (~4 min, ~36 GB RAM)
    python oracle/make_golden.py c5_10      # all 10 C5 cycles (~23 min, ~36 GB RAM)

Floats are stored as float.hex() strings so the fixtures are bit-exact.
"""
from __future__ import annotations

import hashlib
import json
import os
import sys
import time

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, HERE)
from pyoracle import CycleSpec, Reference, SMOOTHERS  # noqa: E402

GOLD = os.path.join(os.path.dirname(HERE), "tests", "golden")


def hx(v):
    return [float(x).hex() for x in np.asarray(v, dtype=np.float64).ravel()]


def sha(v):
    return hashlib.sha256(np.ascontiguousarray(v, dtype=np.float64).tobytes()).hexdigest()


def save(name, obj):
    os.makedirs(GOLD, exist_ok=True)
    with open(os.path.join(GOLD, name + ".json"), "w") as f:
        json.dump(obj, f, indent=1)
    print("wrote", name, flush=True)


def solve_case(name, levels, spec: CycleSpec, coarse=(1, 1), coords="cartesian", alpha=1.0, beta=1.0,
               grading=(1.0, 1.0), seed_f=1, seed_x=0, keep_x=False):
    t0 = time.time()
    ref = Reference(levels, coarse[0], coarse[1], grading, coords, alpha, beta)
    n = ref.n(levels)
    b = Reference.random_vector(n, seed_f)
    x = Reference.random_vector(n, seed_x) if seed_x else np.zeros(n)
    setup = time.time() - t0
    r = ref.solve(spec, b, x)
    obj = dict(
        problem=dict(levels=levels, coarse_nx=coarse[0], coarse_ny=coarse[1], coords=coords,
                     alpha=alpha, beta=beta, grading=list(grading), seed_f=seed_f, seed_x=seed_x),
        spec=spec.__dict__,
        status=r.status, message=r.message, iterations=r.iterations, converged=r.converged,
        history=hx(r.history), history_dec=["%.17e" % h for h in r.history],
        x_sha256=sha(x), x_head=hx(x[:8]), x_tail=hx(x[-8:]),
        ref_wall_seconds=r.wall_seconds, ref_setup_seconds=setup,
        generator="oracle/make_golden.py via oracle/_ref/libgmg_ref_capi.so (reference sources)",
    )
    if keep_x:
        obj["x"] = hx(x)
    save(name, obj)
    del ref
    return obj


def ops_case(name, levels, coarse, coords, alpha, beta, grading):
    """Every per-level operator on seeded inputs, small grids, full vectors."""
    ref = Reference(levels, coarse[0], coarse[1], grading, coords, alpha, beta)
    out = dict(problem=dict(levels=levels, coarse_nx=coarse[0], coarse_ny=coarse[1], coords=coords,
                            alpha=alpha, beta=beta, grading=list(grading)), levels={})
    for l in range(1, levels + 1):
        n = ref.n(l)
        x = Reference.random_vector(n, 100 + l)
        b = Reference.random_vector(n, 200 + l)
        e = dict(shape=list(ref.shapes[l]), x_seed=100 + l, b_seed=200 + l,
                 apply=hx(ref.apply(l, x)), residual=hx(ref.residual(l, x, b)),
                 norm_l2=float(ref.norm_l2(x, l)).hex(), dot=float(ref.dot(x, b, l)).hex())
        sm = {}
        for k in SMOOTHERS:
            om = 1.1 if k in ("jacobi", "richardson", "ilu0") else 0.9
            sm[k] = dict(smoother_omega=om, omega_damp=0.7, out=hx(ref.smooth_step(l, k, om, 0.7, x, b)))
        e["smooth_step"] = sm
        if l >= 2:
            c = Reference.random_vector(ref.n(l - 1), 300 + l)
            e["restriction"] = hx(ref.restriction(l, x))
            e["prolongation"] = dict(c_seed=300 + l, out=hx(ref.prolongation(l - 1, c)))
            e["adaptive_omega"] = float(ref.adaptive_omega(l, b, x)).hex()
        out["levels"][str(l)] = e
    b1 = Reference.random_vector(ref.n(1), 400)
    out["coarse_solve"] = dict(b_seed=400, out=hx(ref.coarse_solve(b1)))
    save(name, out)


START_CASES = [
    # levels, coarse, coords, alpha, grading, smoother, smoother_omega
    (5, (1, 1), "cartesian", 1.0, (1.0, 1.0), "jacobi", 1.0),
    (5, (2, 3), "cylindrical", 0.3, (1.0, 1.0), "gauss_seidel", 1.0),
    (4, (1, 1), "spherical", 1.3, (1.1, 0.93), "adi", 0.9),
    (4, (3, 2), "cartesian", 0.1, (1.0, 1.02), "ilu0", 1.1),
    (4, (1, 1), "cartesian", 1.0, (1.0, 1.0), "richardson", 5.0),
    (1, (5, 4), "cartesian", 1.0, (1.0, 1.0), "sor", 1.3),
]


def start_vectors():
    """gmg::make_start_vector (study.cpp:40-79), nested, on small problems: full vectors."""
    cases = []
    for levels, coarse, coords, alpha, grading, sm, som in START_CASES:
        ref = Reference(levels, coarse[0], coarse[1], grading, coords, alpha, 1.0)
        b = Reference.random_vector(ref.n(levels), 5)
        spec = CycleSpec(smoother=sm, smoother_omega=som, smoothing_omega=0.7)
        cases.append(dict(problem=dict(levels=levels, coarse_nx=coarse[0], coarse_ny=coarse[1], coords=coords,
                                       alpha=alpha, beta=1.0, grading=list(grading)),
                          b_seed=5, spec=spec.__dict__, nested=hx(ref.start_vector(spec, "nested", b))))
    save("start_vectors", dict(cases=cases, generator="oracle/make_golden.py via oracle/_ref (reference sources)"))


def fast():
    rv = Reference.random_vector(64, 1)
    save("random_vector", dict(seed=1, n=64, values=hx(rv)))
    ops_case("ops_cartesian_uniform", 4, (1, 1), "cartesian", 1.0, 1.0, (1.0, 1.0))
    ops_case("ops_cartesian_aniso", 4, (2, 3), "cartesian", 1e-2, 1.0, (1.0, 1.0))
    ops_case("ops_cylindrical", 4, (1, 1), "cylindrical", 1.0, 1.0, (1.0, 1.0))
    ops_case("ops_spherical_graded", 3, (3, 2), "spherical", 1.3, 0.7, (1.1, 0.93))
    jac = lambda **k: CycleSpec(smoother="jacobi", smoother_omega=1.0, smoothing_omega=0.7, **k)
    # C1 (BASELINE configs[0]) adaptive and the fixed omega_l = 4 parity variant
    solve_case("c1_adaptive", 7, jac(tolerance=1e-8), keep_x=True)
    solve_case("c1_fixed4", 7, jac(tolerance=1e-8, adaptive_correction=False, correction_omega=4.0))
    # C3' (cylindrical stand-in for the polar C3), 1023^2
    solve_case("c3p_cylindrical", 10, jac(tolerance=1e-8), coords="cylindrical")
    # small V/W/F variants and edge cases
    solve_case("small_V_jacobi", 6, jac(cycle="V", tolerance=1e-10, max_cycles=40), seed_x=2)
    solve_case("small_W_jacobi", 6, jac(cycle="W", tolerance=1e-10, max_cycles=40), seed_x=2)
    solve_case("small_F_rect_coarse", 5, jac(tolerance=1e-10, pre_steps=3, post_steps=1), coarse=(3, 2),
               alpha=0.1, beta=1.0, seed_x=2)
    solve_case("small_F_graded_sph", 5, jac(tolerance=1e-9), coords="spherical", grading=(1.05, 0.97))
    solve_case("small_F_m0", 6, jac(tolerance=1e-9, pre_steps=0, post_steps=3))
    solve_case("small_F_n0", 6, jac(tolerance=1e-9, pre_steps=3, post_steps=0))
    solve_case("small_F_coarse_cap", 6, jac(tolerance=1e-9, coarse_direct_max_neq=0), coarse=(3, 3))
    solve_case("single_level", 1, jac(tolerance=1e-12), coarse=(5, 4))
    solve_case("diverge_omega", 6, jac(tolerance=1e-12, adaptive_correction=False, correction_omega=40.0,
                                       max_cycles=30))
    solve_case("c4_small_2047", 11, jac(tolerance=1e-10, max_cycles=3))
    start_vectors()


def c4():
    jac = CycleSpec(smoother="jacobi", smoothing_omega=0.7, tolerance=1e-10)
    solve_case("c4_adaptive", 13, jac)


def c2():
    for eps in (1.0, 1e-1, 1e-2, 1e-3):
        for s in (1, 2, 4):
            spec = CycleSpec(smoother="gauss_seidel", smoother_omega=1.0, smoothing_omega=0.7,
                             pre_steps=s, post_steps=s, tolerance=1e-8, max_cycles=50)
            solve_case(f"c2_eps{eps:g}_s{s}", 10, spec, alpha=eps, beta=1.0, seed_x=2)


def c5():
    spec = CycleSpec(smoother="jacobi", smoothing_omega=0.7, pre_steps=3, post_steps=3,
                     tolerance=1e-30, max_cycles=1)
    solve_case("c5_1cycle", 14, spec, alpha=1e-2, beta=1.0, seed_x=2)


def c5_10():
    """BASELINE config 5 exactly: 10 F-cycles (tol=1e-30, max_cycles=10, the reference's
    fixed-budget idiom, tests/test_study.cpp:112-113). ~23 min of CPU, ~36 GB RAM."""
    spec = CycleSpec(smoother="jacobi", smoothing_omega=0.7, pre_steps=3, post_steps=3,
                     tolerance=1e-30, max_cycles=10)
    solve_case("c5_10cycle", 14, spec, alpha=1e-2, beta=1.0, seed_x=2)


if __name__ == "__main__":
    if not Reference.available():
        sys.exit("oracle/_ref not built: run make -C oracle where /root/reference exists")
    what = sys.argv[1:] or ["fast"]
    for w in what:
        globals()[w]()
