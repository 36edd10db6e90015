"""Parity of the CUDA path (through the C ABI, libgmg_b200.so) with the CPU
oracle and the reference's golden fixtures. The bar is bit-for-bit identity of
every grid function, every residual history and every iteration count (the
arithmetic is fp64 in the reference's operation order);
the only tolerance used anywhere is for the opt-in "fast" reduction mode.
"""
import numpy as np
import pytest

from conftest import bits_equal, first_mismatch, load_golden, unhex
from pyoracle import CycleSpec as OSpec
from pyoracle import Oracle

gmg = pytest.importorskip("paper_0805_3041_b200.gmg")

pytestmark = pytest.mark.gpu

GEOMS = [
    dict(levels=5, coarse=(1, 1), coords="cartesian", alpha=1.0, beta=1.0, grading=(1.0, 1.0)),
    dict(levels=4, coarse=(2, 3), coords="cartesian", alpha=1e-2, beta=1.0, grading=(1.0, 1.0)),
    dict(levels=5, coarse=(1, 1), coords="cylindrical", alpha=1.0, beta=1.0, grading=(1.0, 1.0)),
    dict(levels=4, coarse=(3, 2), coords="spherical", alpha=1.3, beta=0.7, grading=(1.1, 0.93)),
    dict(levels=3, coarse=(60, 1), coords="cartesian", alpha=0.5, beta=2.0, grading=(1.0, 1.02)),
]
GIDS = ["cart_uniform", "cart_aniso_rect", "cylindrical", "spherical_graded", "wide_graded"]


def pair(geom):
    args = (geom["levels"], geom["coarse"][0], geom["coarse"][1], geom["grading"], geom["coords"],
            geom["alpha"], geom["beta"])
    return gmg.MultilevelProblem(*args), Oracle(*args)


@pytest.fixture(scope="module")
def problems(gpu):
    return [pair(g) for g in GEOMS]


def test_operator_classes(problems):
    kinds = [p.coef_kind(p.num_levels) for p, _ in problems]
    assert kinds[0] == "const"  # dyadic uniform grid: bit-exact constant stencil
    assert kinds[1] in ("const", "rowx", "field", "axes")  # 23 x 31 cells: h = 1/24 is not dyadic
    assert kinds[2] == "rowx"
    assert kinds[3] == "axes"  # graded spherical: rebuilt on the fly from 1-D tables (0 B/DOF)


@pytest.mark.parametrize("gi", [3, 4], ids=["spherical_graded", "wide_graded"])
def test_axes_and_field_storage_agree(problems, gi):
    """The same graded operator stored as five streamed arrays (FIELD: built from the
    arrays alone, without the physics) and computed on the fly (AXES): every level's
    smoother and whole solves bit for bit (stencil.cpp:77-127)."""
    d, o = problems[gi]
    levels = [dict(nx=o.shapes[l][0], ny=o.shapes[l][1], **dict(zip(("x", "y"), o.coords(l))), **o.operator(l))
              for l in range(1, d.num_levels + 1)]
    f = gmg.MultilevelProblem.from_levels(levels)
    L = d.num_levels
    assert f.coef_kind(L) == "field" and d.coef_kind(L) == "axes"
    x = Oracle.random_vector(d.n(L), 5)
    b = Oracle.random_vector(d.n(L), 6)
    for l in range(1, L + 1):
        xl, bl = Oracle.random_vector(d.n(l), 7), Oracle.random_vector(d.n(l), 8)
        assert bits_equal(gmg.smooth_step(d, l, "jacobi", 1.0, xl, bl, 0.7), gmg.smooth_step(f, l, "jacobi", 1.0, xl, bl, 0.7))
        assert bits_equal(gmg.apply(d, l, xl), gmg.apply(f, l, xl))
    spec = gmg.CycleSpec(smoother="jacobi", tolerance=1e-9, max_cycles=20)
    xa, xf = x.copy(), x.copy()
    ra, rf = gmg.solve(d, b, spec, xa), gmg.solve(f, b, spec, xf)
    assert ra.residual_history == rf.residual_history and bits_equal(xa, xf)


@pytest.mark.parametrize("gi", range(len(GEOMS)), ids=GIDS)
def test_per_level_operators_bitexact(problems, gi):
    d, o = problems[gi]
    for l in range(1, d.num_levels + 1):
        n = d.n(l)
        x = Oracle.random_vector(n, 10 + l)
        b = Oracle.random_vector(n, 20 + l)
        assert bits_equal(gmg.apply(d, l, x), o.apply(l, x)), ("apply", l)
        assert bits_equal(gmg.residual(d, l, x, b), o.residual(l, x, b)), ("residual", l)
        for kind, som in (("jacobi", 1.0), ("jacobi", 1.3), ("gauss_seidel", 1.0), ("sor", 1.4), ("sor", 0.6)):
            for damp in (0.7, 1.0, 0.35):
                got = gmg.smooth_step(d, l, kind, som, x, b, damp)
                want = o.smooth_step(l, kind, som, damp, x, b)
                assert bits_equal(got, want), ("smooth_step", kind, som, l, damp, first_mismatch(got, want))
        if l >= 2:
            assert bits_equal(gmg.restriction(d, l, x), o.restriction(l, x)), ("restriction", l)
            c = Oracle.random_vector(d.n(l - 1), 30 + l)
            assert bits_equal(gmg.prolongation(d, l - 1, c), o.prolongation(l - 1, c)), ("prolongation", l)
            # defect/correction pairs as the cycle produces them, and random ones
            corr = o.prolongation(l - 1, c)
            assert gmg.adaptive_omega(d, l, b, corr) == o.adaptive_omega(l, b, corr)
            assert gmg.adaptive_omega(d, l, b, x * x) == o.adaptive_omega(l, b, x * x)
        assert gmg.norm_l2(d, x) == o.norm_l2(x)
        assert gmg.dot(d, x, b) == o.dot(x, b)
    b1 = Oracle.random_vector(d.n(1), 5)
    assert bits_equal(gmg.coarse_solve(d, b1), o.coarse_solve(b1))


def test_adaptive_omega_zero_correction_is_one(problems):
    d, _ = problems[0]
    l = d.num_levels
    assert gmg.adaptive_omega(d, l, np.ones(d.n(l)), np.zeros(d.n(l))) == 1.0


def oracle_levels(o):
    out = []
    for l in range(1, o.levels + 1):
        nx, ny = o.shapes[l]
        x, y = o.coords(l)
        out.append(dict(nx=nx, ny=ny, x=x, y=y, **o.operator(l)))
    return out


def test_problem_from_reference_arrays_matches_host_assembly(gpu):
    """The generic C-ABI descriptor path (the five StencilOperator arrays per level, as the
    C++ shim passes a reference MultilevelProblem) gives the same solve as host assembly."""
    o = Oracle(6, 1, 2, (1.02, 1.0), "cylindrical", 0.3, 1.0)
    d1 = gmg.MultilevelProblem.from_levels(oracle_levels(o))
    d2 = gmg.MultilevelProblem(6, 1, 2, (1.02, 1.0), "cylindrical", 0.3, 1.0)
    n = d1.n(6)
    b = gmg.random_vector(n, 1)
    spec = gmg.CycleSpec(smoother="jacobi", tolerance=1e-10)
    x1, x2, xo = np.zeros(n), np.zeros(n), np.zeros(n)
    r1, r2 = gmg.solve(d1, b, spec, x1), gmg.solve(d2, b, spec, x2)
    ro = o.solve(OSpec(smoother="jacobi", tolerance=1e-10), b, xo)
    assert bits_equal(r1.residual_history, ro.history) and bits_equal(r2.residual_history, ro.history)
    assert bits_equal(x1, xo) and bits_equal(x2, xo)


def test_adaptive_omega_nonpositive_energy_raises(gpu):
    # cycle.cpp:48-49: (A c, c) <= 0 throws runtime_error. Use an indefinite finest operator.
    o = Oracle(3)
    lv = oracle_levels(o)
    lv[2]["c"] = -lv[2]["c"]
    d = gmg.MultilevelProblem.from_levels(lv)
    n = d.n(3)
    with pytest.raises(gmg.GmgRuntimeError, match="nonpositive energy"):
        gmg.adaptive_omega(d, 3, np.ones(n), gmg.random_vector(n, 3))
    # and through a solve: the reference aborts the solve with the same error
    with pytest.raises(gmg.GmgRuntimeError, match="nonpositive energy"):
        gmg.solve(d, gmg.random_vector(n, 1), gmg.CycleSpec(smoother="jacobi"), np.zeros(n))


@pytest.mark.parametrize("n", [1, 31, 8192, 8193, 100003, 1 << 20])
def test_exact_dot_and_norm_on_device(problems, n):
    d, o = problems[0]
    if n > d.n(d.num_levels) * 1:
        d = gmg.MultilevelProblem(11)
    rng = np.random.default_rng(n)
    for a, b in [(rng.uniform(-1, 1, n), rng.uniform(-1, 1, n)),
                 (np.ldexp(np.round(rng.uniform(-8, 8, n)), -rng.integers(0, 4, n)), np.ones(n)),
                 (rng.uniform(-1, 1, n) * 10.0 ** rng.integers(-12, 12, n), rng.uniform(0, 1, n))]:
        assert gmg.dot(d, a, b) == o.dot(a, b)
        assert gmg.norm_l2(d, a) == o.norm_l2(a)
        assert abs(gmg.dot(d, a, b, reduction="fast") - o.dot(a, b)) <= 1e-10 * (np.abs(a * b).sum() + 1e-300)


def test_exact_sums_failed_speculation_and_literal_chunks(gpu):
    """Inputs that defeat the walk's speculation (the approximate prefix lands in another
    binade than the sequential sum) and chunks too dense in breaks to record: the chain must
    fall back to literal re-sums and still return the left-to-right result bit for bit
    (stencil.cpp:9-26). The engine counters prove the fallback paths ran."""
    d = gmg.MultilevelProblem(11)
    o = Oracle(3)
    n = 1 << 20
    rng = np.random.default_rng(5)
    cancel = rng.uniform(-1, 1, n)
    cancel[::4096] = 1e17
    cancel[1::4096] = -1e17
    spike = np.full(n, 2.0 ** -30)
    spike[n // 3] = 2.0 ** 40
    spike[2 * n // 3] = -2.0 ** 40
    alternating = np.where(np.arange(n) % 2 == 0, 1.0, -1.0) * (1 + 2.0 ** -30 * rng.integers(0, 8, n))
    ones = np.ones(n)
    for name, a, want_dense in (("cancel", cancel, False), ("spike", spike, True), ("alternating", alternating, True)):
        gmg.seqsum_stats(d, reset=True)
        assert gmg.dot(d, a, ones) == o.dot(a, ones), name
        assert gmg.norm_l2(d, a) == o.norm_l2(a), name
        st = gmg.seqsum_stats(d)
        assert st["rewalks"] > 0, (name, st)
        if want_dense:
            assert st["dense_chunks"] > 0, (name, st)


def test_axpy(problems):
    d, _ = problems[0]
    x = Oracle.random_vector(1000, 1)
    y = Oracle.random_vector(1000, 2)
    want = y + 0.3 * x
    gmg.axpy(d, 0.3, x, y)
    assert bits_equal(y, want)


@pytest.mark.parametrize("smoother", ["jacobi", "gauss_seidel"])
@pytest.mark.parametrize("cycle", ["V", "W"])
@pytest.mark.parametrize("gi", [0, 2, 3], ids=["cart", "cyl", "sph"])
def test_mg_cycle_bitexact(problems, cycle, gi, smoother):
    d, o = problems[gi]
    L = d.num_levels
    for adaptive in (True, False):
        spec = dict(cycle=cycle, smoother=smoother, pre_steps=2, post_steps=1, adaptive_correction=adaptive,
                    correction_omega=3.0)
        for l in range(1, L + 1):
            u0 = Oracle.random_vector(d.n(l), 40 + l)
            g = Oracle.random_vector(d.n(l), 50 + l)
            got = gmg.mg_cycle(d, l, u0, g, gmg.CycleSpec(**spec))
            want = o.mg_cycle(OSpec(**spec), l, u0, g)
            assert bits_equal(got, want), (cycle, l, adaptive, first_mismatch(got, want))


SOLVE_FIXTURES = ["c1_adaptive", "c1_fixed4", "small_V_jacobi", "small_W_jacobi", "small_F_rect_coarse",
                  "small_F_graded_sph", "small_F_m0", "small_F_n0", "small_F_coarse_cap", "single_level",
                  "c3p_cylindrical", "c4_small_2047"]


def run_fixture(name, spec_over=None):
    g = load_golden(name)
    pb = g["problem"]
    d = gmg.MultilevelProblem(pb["levels"], pb["coarse_nx"], pb["coarse_ny"], tuple(pb["grading"]),
                              pb["coords"], pb["alpha"], pb["beta"])
    L = pb["levels"]
    n = d.n(L)
    b = gmg.random_vector(n, pb["seed_f"])
    x = gmg.random_vector(n, pb["seed_x"]) if pb["seed_x"] else np.zeros(n)
    spec = dict(g["spec"])
    spec.update(spec_over or {})
    return g, d, b, x, gmg.CycleSpec(**spec)


@pytest.mark.parametrize("name", SOLVE_FIXTURES)
def test_solve_matches_reference_golden(gpu, name):
    g, d, b, x, spec = run_fixture(name)
    rep = gmg.solve(d, b, spec, x)
    want = unhex(g["history"])
    assert rep.iterations == g["iterations"]
    assert rep.converged == g["converged"]
    assert bits_equal(rep.residual_history, want), first_mismatch(rep.residual_history, want)
    assert bits_equal(x[:8], unhex(g["x_head"])) and bits_equal(x[-8:], unhex(g["x_tail"]))
    if "x" in g:
        assert bits_equal(x, unhex(g["x"]))
    # SolveReport invariants (test_cycle.cpp:214-231)
    h = rep.residual_history
    assert len(h) == rep.iterations + 1 and len(rep.convergence_factors) == rep.iterations
    for k, f in enumerate(rep.convergence_factors):
        assert f == h[k + 1] / h[k]


def test_solve_divergence_error_carries_report(gpu):
    g, d, b, x, spec = run_fixture("diverge_omega")
    with pytest.raises(gmg.DivergenceError) as ei:
        gmg.solve(d, b, spec, x)
    rep = ei.value.report
    assert rep.iterations == g["iterations"] and not rep.converged
    assert bits_equal(rep.residual_history, unhex(g["history"]))
    assert "grew beyond 1e6" in str(ei.value)
    assert bits_equal(x[:8], unhex(g["x_head"]))


def test_solve_errors_match_reference(gpu):
    d = gmg.MultilevelProblem(3)
    b = gmg.random_vector(d.n(3), 1)
    with pytest.raises(gmg.InvalidArgument, match="smoother_omega"):
        gmg.solve(d, b, gmg.CycleSpec(smoother="jacobi", smoother_omega=0.0), np.zeros(d.n(3)))
    with pytest.raises(gmg.InvalidArgument, match="pre_steps/post_steps"):
        gmg.solve(d, b, gmg.CycleSpec(smoother="jacobi", pre_steps=0, post_steps=0), np.zeros(d.n(3)))
    with pytest.raises(gmg.InvalidArgument, match="omega: damping"):
        gmg.solve(d, b, gmg.CycleSpec(smoother="jacobi", smoothing_omega=0.0), np.zeros(d.n(3)))
    with pytest.raises(gmg.LogicError):
        gmg.solve(d, b[:-1], gmg.CycleSpec(smoother="jacobi"), np.zeros(d.n(3)))
    # zero right-hand side and zero start: converged at cycle 0 (cycle.cpp:164-170)
    rep = gmg.solve(d, np.zeros(d.n(3)), gmg.CycleSpec(smoother="jacobi"), np.zeros(d.n(3)))
    assert rep.converged and rep.iterations == 0 and rep.residual_history == [0.0]


def test_fast_reduction_mode_close(gpu):
    g, d, b, x, spec = run_fixture("c1_adaptive", {"reduction": "fast"})
    rep = gmg.solve(d, b, spec, x)
    want = unhex(g["history"])
    assert rep.iterations == g["iterations"]
    np.testing.assert_allclose(rep.residual_history, want, rtol=1e-6)


def test_repeated_solves_are_deterministic(gpu):
    g, d, b, x0, spec = run_fixture("c3p_cylindrical")
    hs = []
    for _ in range(2):
        x = x0.copy()
        hs.append(gmg.solve(d, b, spec, x).residual_history)
    assert bits_equal(hs[0], hs[1])


C2_FIXTURES = [f"c2_eps{e}_s{k}" for e in ("1", "0.1", "0.01", "0.001") for k in (1, 2, 4)]


@pytest.mark.parametrize("name", C2_FIXTURES)
def test_c2_gauss_seidel_matches_reference_golden(gpu, name):
    """BASELINE configs[1]: anisotropic -eps u_xx - u_yy on 1023^2 (10 levels), random start,
    lexicographic Gauss-Seidel s+s, adaptive omega_l, up to 50 cycles — bit for bit."""
    g, d, b, x, spec = run_fixture(name)
    rep = gmg.solve(d, b, spec, x)
    want = unhex(g["history"])
    assert rep.iterations == g["iterations"] and rep.converged == g["converged"]
    assert bits_equal(rep.residual_history, want), first_mismatch(rep.residual_history, want)
    assert bits_equal(x[:8], unhex(g["x_head"])) and bits_equal(x[-8:], unhex(g["x_tail"]))


@pytest.mark.parametrize("smoother,som", [("gauss_seidel", 1.0), ("sor", 1.3)])
@pytest.mark.parametrize("cycle", ["V", "W", "F"])
def test_gs_solves_bitexact_vs_oracle(gpu, smoother, som, cycle):
    for coords, grading, coarse in (("cartesian", (1.0, 1.0), (1, 1)), ("spherical", (1.05, 0.97), (2, 3))):
        args = (5, coarse[0], coarse[1], grading, coords, 0.3, 1.0)
        d, o = gmg.MultilevelProblem(*args), Oracle(*args)
        n = d.n(5)
        b = gmg.random_vector(n, 1)
        x0 = gmg.random_vector(n, 2)
        kw = dict(cycle=cycle, smoother=smoother, smoother_omega=som, pre_steps=2, post_steps=3, tolerance=1e-11,
                  max_cycles=30)
        xg, xo = x0.copy(), x0.copy()
        rg = gmg.solve(d, b, gmg.CycleSpec(**kw), xg)
        ro = o.solve(OSpec(**kw), b, xo)
        assert rg.iterations == ro.iterations and bits_equal(rg.residual_history, ro.history)
        assert bits_equal(xg, xo)


@pytest.mark.slow
def test_c5_full_size_first_cycle(gpu):
    """BASELINE configs[4] at full size (16383^2 interior, 14 levels, eps=1e-2, jacobi 3+3, random
    start): the reference's first F-cycle (r0, r1) and solution, bit for bit."""
    g, d, b, x, spec = run_fixture("c5_1cycle")
    rep = gmg.solve(d, b, spec, x)
    assert rep.iterations == 1
    assert bits_equal(rep.residual_history, unhex(g["history"])), \
        first_mismatch(rep.residual_history, unhex(g["history"]))
    assert bits_equal(x[:8], unhex(g["x_head"])) and bits_equal(x[-8:], unhex(g["x_tail"]))
    import hashlib
    assert hashlib.sha256(np.ascontiguousarray(x).tobytes()).hexdigest() == g["x_sha256"]


@pytest.mark.slow
def test_c4_full_size_history(gpu):
    """BASELINE configs[3] at full size (8191^2 interior, 13 levels): the
    reference's 12-cycle history, bit for bit."""
    g, d, b, x, spec = run_fixture("c4_adaptive")
    rep = gmg.solve(d, b, spec, x)
    assert rep.iterations == g["iterations"] == 12
    assert bits_equal(rep.residual_history, unhex(g["history"])), \
        first_mismatch(rep.residual_history, unhex(g["history"]))
    assert bits_equal(x[:8], unhex(g["x_head"])) and bits_equal(x[-8:], unhex(g["x_tail"]))
    import hashlib
    assert hashlib.sha256(np.ascontiguousarray(x).tobytes()).hexdigest() == g["x_sha256"]


@pytest.mark.slow
def test_c5_full_size_ten_cycles(gpu):
    """BASELINE configs[4] exactly: 10 F-cycles (tol=1e-30, max_cycles=10, the reference's
    fixed-budget idiom): all 11 residuals and the final solution, bit for bit."""
    g, d, b, x, spec = run_fixture("c5_10cycle")
    rep = gmg.solve(d, b, spec, x)
    assert rep.iterations == g["iterations"] == 10
    assert bits_equal(rep.residual_history, unhex(g["history"])), \
        first_mismatch(rep.residual_history, unhex(g["history"]))
    import hashlib
    assert hashlib.sha256(np.ascontiguousarray(x).tobytes()).hexdigest() == g["x_sha256"]


@pytest.mark.parametrize("alpha", [1.0, 1e-2, 0.3])
def test_jacobi_division_paths_edge_values(gpu, alpha):
    """The Jacobi preconditioner z = d / c (smoother.cpp:293-295) on the warp-strip
    kernels: exact reciprocal (c = 4), the reciprocal-FMA path with its out-of-range
    fallback (c = 2 + 2 alpha), on defects spanning zeros of both signs, subnormals,
    tiny and huge magnitudes; M = 1..4 fused steps; bit for bit against the oracle."""
    levels = 9  # 511^2: k_smooth4
    a = (levels, 1, 1, (1.0, 1.0), "cartesian", alpha, 1.0)
    d, o = gmg.MultilevelProblem(*a), Oracle(*a)
    n = d.n(levels)
    rng = np.random.default_rng(7)
    mags = np.array([0.0, -0.0, 5e-324, 1e-310, 1e-300, 2.0 ** -960, 2.0 ** -959, 1e-12, 1.0, 1e12, 2.0 ** 959,
                     2.0 ** 960, 1e300])
    x = rng.choice(mags, n) * rng.choice([-1.0, 1.0], n)
    b = rng.choice(mags, n) * rng.choice([-1.0, 1.0], n)
    x[: n // 2] = Oracle.random_vector(n // 2, 3)  # half ordinary values
    for damp in (0.7, 1.0):
        got = gmg.smooth_step(d, levels, "jacobi", 1.0, x, b, damp)
        want = o.smooth_step(levels, "jacobi", 1.0, damp, x, b)
        assert bits_equal(got, want), (damp, first_mismatch(got, want))
    # fused steps (mg_cycle's pre-smoothing from u) on ordinary data
    xo = Oracle.random_vector(n, 4)
    bo = Oracle.random_vector(n, 5)
    for steps in (2, 3, 4):
        spec = dict(cycle="V", smoother="jacobi", pre_steps=steps, post_steps=0)
        got = gmg.mg_cycle(d, levels, xo, bo, gmg.CycleSpec(**spec))
        want = o.mg_cycle(OSpec(**spec), levels, xo, bo)
        assert bits_equal(got, want), (steps, first_mismatch(got, want))


def test_pageable_vectors_staged_like_pinned(gpu):
    """gmg_dev_solve takes pageable host vectors (the shim's std::vector storage) through the
    pinned staging ring (solver.cu staged_rows, vectors >= 32 MB) and pinned ones straight to
    the copy engine: same history and the same x, bit for bit, on a rectangular grid whose
    rows do not fill the last chunk; the random start vector travels in, so both directions
    are covered."""
    import torch
    d = gmg.MultilevelProblem(8, 19, 13, (1.0, 1.0), "cartesian", 1.0, 0.3)
    n = d.n(8)
    assert n * 8 >= 32 << 20
    b = gmg.random_vector(n, 5)
    x0 = gmg.random_vector(n, 6)
    spec = gmg.CycleSpec(tolerance=1e-6, max_cycles=3, smoother="jacobi", smoothing_omega=0.7,
                         pre_steps=1, post_steps=1, cycle="F", adaptive_correction=True)
    xs = x0.copy()
    rs = gmg.solve(d, b, spec, xs)
    pb = torch.from_numpy(b).pin_memory()
    px = torch.from_numpy(x0.copy()).pin_memory()
    rp = gmg.solve(d, pb.numpy(), spec, px.numpy())
    assert bits_equal(rs.residual_history, rp.residual_history)
    assert bits_equal(xs, px.numpy())
    # zero cycles: x comes back exactly as it went in
    xr = x0.copy()
    gmg.solve(d, b, gmg.CycleSpec(tolerance=1e-6, max_cycles=0, smoother="jacobi", smoothing_omega=0.7), xr)
    assert bits_equal(xr, x0)
