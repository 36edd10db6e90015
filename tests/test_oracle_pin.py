"""Pins the CPU oracle (oracle/gmg_oracle.c, a C restatement of the reference
path) before it is trusted as the parity checker:
  * against golden fixtures produced by the reference itself (tests/golden/,
    oracle/make_golden.py), bit for bit;
  * against the compiled reference (oracle/_ref) on randomized cases, when the
    reference build is present.
CPU only."""
import numpy as np
import pytest

from conftest import bits_equal, first_mismatch, load_golden, unhex
from pyoracle import SMOOTHERS, CycleSpec, Oracle, Reference

OPS_FIXTURES = ["ops_cartesian_uniform", "ops_cartesian_aniso", "ops_cylindrical", "ops_spherical_graded"]
SOLVE_FIXTURES = ["c1_adaptive", "c1_fixed4", "small_V_jacobi", "small_W_jacobi", "small_F_rect_coarse",
                  "small_F_graded_sph", "small_F_m0", "small_F_n0", "small_F_coarse_cap", "single_level",
                  "diverge_omega", "c3p_cylindrical", "c4_small_2047"]


def make(problem, cls=Oracle):
    return cls(problem["levels"], problem["coarse_nx"], problem["coarse_ny"], tuple(problem["grading"]),
               problem["coords"], problem["alpha"], problem["beta"])


def test_random_vector_matches_libstdcxx():
    g = load_golden("random_vector")
    assert bits_equal(Oracle.random_vector(g["n"], g["seed"]), unhex(g["values"]))


@pytest.mark.parametrize("name", OPS_FIXTURES)
def test_oracle_operators_match_reference_golden(name):
    g = load_golden(name)
    o = make(g["problem"])
    for ls, e in g["levels"].items():
        l = int(ls)
        x = Oracle.random_vector(o.n(l), e["x_seed"])
        b = Oracle.random_vector(o.n(l), e["b_seed"])
        assert bits_equal(o.apply(l, x), unhex(e["apply"])), (l, "apply")
        assert bits_equal(o.residual(l, x, b), unhex(e["residual"])), (l, "residual")
        assert o.norm_l2(x) == unhex(e["norm_l2"])
        assert o.dot(x, b) == unhex(e["dot"])
        for k, s in e["smooth_step"].items():
            got = o.smooth_step(l, k, s["smoother_omega"], s["omega_damp"], x, b)
            assert bits_equal(got, unhex(s["out"])), (l, k, first_mismatch(got, unhex(s["out"])))
        if l >= 2:
            assert bits_equal(o.restriction(l, x), unhex(e["restriction"])), (l, "restriction")
            c = Oracle.random_vector(o.n(l - 1), e["prolongation"]["c_seed"])
            assert bits_equal(o.prolongation(l - 1, c), unhex(e["prolongation"]["out"])), (l, "prolongation")
            assert o.adaptive_omega(l, b, x) == unhex(e["adaptive_omega"])
    b1 = Oracle.random_vector(o.n(1), g["coarse_solve"]["b_seed"])
    assert bits_equal(o.coarse_solve(b1), unhex(g["coarse_solve"]["out"]))


@pytest.mark.parametrize("name", SOLVE_FIXTURES)
def test_oracle_solve_matches_reference_golden(name):
    g = load_golden(name)
    o = make(g["problem"])
    L = g["problem"]["levels"]
    n = o.n(L)
    b = Oracle.random_vector(n, g["problem"]["seed_f"])
    x = Oracle.random_vector(n, g["problem"]["seed_x"]) if g["problem"]["seed_x"] else np.zeros(n)
    r = o.solve(CycleSpec(**g["spec"]), b, x)
    assert r.status == g["status"]
    assert r.iterations == g["iterations"]
    assert r.converged == g["converged"]
    assert bits_equal(r.history, unhex(g["history"]))
    assert bits_equal(x[:8], unhex(g["x_head"])) and bits_equal(x[-8:], unhex(g["x_tail"]))
    if "x" in g:
        assert bits_equal(x, unhex(g["x"]))


needs_ref = pytest.mark.skipif(not Reference.available(), reason="oracle/_ref (compiled reference) not built")


@needs_ref
@pytest.mark.parametrize("coords", ["cartesian", "cylindrical", "spherical"])
def test_oracle_vs_reference_randomized(coords):
    rng = np.random.default_rng(hash(coords) % 2**32)
    for trial in range(3):
        levels = int(rng.integers(2, 5))
        cnx, cny = int(rng.integers(1, 4)), int(rng.integers(1, 4))
        grading = (float(rng.uniform(0.9, 1.1)), float(rng.uniform(0.9, 1.1)))
        a, bb = float(rng.uniform(0.01, 2)), float(rng.uniform(0.01, 2))
        o = Oracle(levels, cnx, cny, grading, coords, a, bb)
        r = Reference(levels, cnx, cny, grading, coords, a, bb)
        for l in range(1, levels + 1):
            x = Oracle.random_vector(o.n(l), 7 + trial)
            b = Oracle.random_vector(o.n(l), 9 + trial)
            for k in "cnsew":
                assert bits_equal(o.operator(l)[k], r.operator(l)[k])
            assert bits_equal(o.apply(l, x), r.apply(l, x))
            for k in SMOOTHERS:
                om = 1.3 if k in ("jacobi", "richardson", "ilu0") else 0.8
                assert bits_equal(o.smooth_step(l, k, om, 0.6, x, b), r.smooth_step(l, k, om, 0.6, x, b)), k
            if l >= 2:
                assert bits_equal(o.restriction(l, x), r.restriction(l, x))
                c = Oracle.random_vector(o.n(l - 1), 3)
                assert bits_equal(o.prolongation(l - 1, c), r.prolongation(l - 1, c))
        for cyc in "VWF":
            spec = CycleSpec(cycle=cyc, smoother="jacobi", tolerance=1e-9, max_cycles=25)
            b = Oracle.random_vector(o.n(levels), 1)
            xo = Oracle.random_vector(o.n(levels), 2)
            xr = xo.copy()
            ro, rr = o.solve(spec, b, xo), r.solve(spec, b, xr)
            assert ro.status == rr.status and ro.iterations == rr.iterations
            assert bits_equal(ro.history, rr.history) and bits_equal(xo, xr)


@needs_ref
def test_oracle_errors_match_reference():
    o, r = Oracle(3), Reference(3)
    b = Oracle.random_vector(o.n(3), 1)
    for spec in [CycleSpec(smoother="gauss_seidel", smoother_omega=2.5),
                 CycleSpec(smoother="jacobi", pre_steps=0, post_steps=0),
                 CycleSpec(smoother="jacobi", smoothing_omega=-1.0),
                 CycleSpec(smoother="tri_x", smoother_omega=1.5)]:
        ro = o.solve(spec, b, np.zeros(o.n(3)))
        rr = r.solve(spec, b, np.zeros(o.n(3)))
        assert ro.status == rr.status != 0
        assert ro.message == rr.message


def test_oracle_start_vector_matches_reference_golden():
    """make_start_vector nested (study.cpp:46-58) for 6 smoothers / 3 coordinate systems."""
    g = load_golden("start_vectors")
    for case in g["cases"]:
        o = make(case["problem"])
        b = Oracle.random_vector(o.n(case["problem"]["levels"]), case["b_seed"])
        got = o.start_vector(CycleSpec(**case["spec"]), "nested", b)
        assert bits_equal(got, unhex(case["nested"])), (case["spec"]["smoother"], first_mismatch(got, unhex(case["nested"])))


@needs_ref
@pytest.mark.parametrize("coords", ["cartesian", "cylindrical", "spherical"])
def test_oracle_start_vector_vs_reference(coords):
    for levels, cn, sm, som in [(6, (1, 1), "jacobi", 1.0), (5, (2, 1), "sor", 1.2), (4, (1, 3), "tri_y", 0.8),
                                (4, (1, 1), "gstri_x", 1.0), (1, (3, 3), "jacobi", 1.0)]:
        o = Oracle(levels, cn[0], cn[1], (1.0, 1.0), coords, 0.05, 1.0)
        r = Reference(levels, cn[0], cn[1], (1.0, 1.0), coords, 0.05, 1.0)
        b = Oracle.random_vector(o.n(levels), 11)
        spec = CycleSpec(smoother=sm, smoother_omega=som, smoothing_omega=0.6)
        for kind in ("zero", "nested"):
            assert bits_equal(o.start_vector(spec, kind, b), r.start_vector(spec, kind, b)), (levels, sm, kind)
    # the reference's errors: damping checked by smooth_step, smoother omega by setup
    o = Oracle(3)
    r = Reference(3)
    b = Oracle.random_vector(o.n(3), 1)
    for spec in (CycleSpec(smoother="jacobi", smoothing_omega=0.0), CycleSpec(smoother="sor", smoother_omega=2.5)):
        with pytest.raises(Exception) as eo:
            o.start_vector(spec, "nested", b)
        with pytest.raises(Exception) as er:
            r.start_vector(spec, "nested", b)
        assert eo.value.code == er.value.code == 2 and eo.value.msg == er.value.msg
