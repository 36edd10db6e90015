"""BASELINE config 3, Poisson in polar coordinates (r in [0.1, 1] Dirichlet,
theta periodic), on the device: every per-level operator, mg_cycle, whole
solves and the full 1023 x 1024 C3 history, bit for bit against the oracle's
restatement (oracle/gmg_oracle.c, CS_POLAR). The reference has no polar
coordinates, so this parity is unpinned by construction; the
oracle's own periodic logic is checked by tests/test_polar_oracle.py."""
import numpy as np
import pytest

from conftest import bits_equal, first_mismatch
from pyoracle import CycleSpec as OSpec
from pyoracle import Oracle

gmg = pytest.importorskip("paper_0805_3041_b200.gmg")

pytestmark = pytest.mark.gpu

GEOMS = {
    "L5_c2": (5, 1, 2, (1.0, 1.0), "polar", 1.0, 1.0),
    "L4_rect_graded": (4, 2, 3, (1.05, 1.0), "polar", 0.5, 2.0),
    "L9_wide": (9, 1, 2, (1.0, 1.0), "polar", 1.0, 1.0),  # 511 x 512: streaming kernels, several row segments
}


@pytest.fixture(scope="module")
def problems(gpu):
    return {k: (gmg.MultilevelProblem(*a), Oracle(*a)) for k, a in GEOMS.items()}


@pytest.mark.parametrize("gi", list(GEOMS))
def test_polar_operators_bitexact(problems, gi):
    d, o = problems[gi]
    for l in range(1, d.num_levels + 1):
        n = d.n(l)
        x = Oracle.random_vector(n, 10 + l)
        b = Oracle.random_vector(n, 20 + l)
        assert bits_equal(gmg.apply(d, l, x), o.apply(l, x)), ("apply", l)
        assert bits_equal(gmg.residual(d, l, x, b), o.residual(l, x, b)), ("residual", l)
        for kind, som, damp in (("jacobi", 1.0, 0.7), ("jacobi", 1.3, 1.0), ("richardson", 0.5, 0.7)):
            got = gmg.smooth_step(d, l, kind, som, x, b, damp)
            want = o.smooth_step(l, kind, som, damp, x, b)
            assert bits_equal(got, want), ("smooth_step", kind, l, first_mismatch(got, want))
        if l >= 2:
            assert bits_equal(gmg.restriction(d, l, x), o.restriction(l, x)), ("restriction", l)
            c = Oracle.random_vector(d.n(l - 1), 30 + l)
            assert bits_equal(gmg.prolongation(d, l - 1, c), o.prolongation(l - 1, c)), ("prolongation", l)
            assert gmg.adaptive_omega(d, l, b, x) == o.adaptive_omega(l, b, x), ("adaptive_omega", l)
    b1 = Oracle.random_vector(d.n(1), 5)
    assert bits_equal(gmg.coarse_solve(d, b1), o.coarse_solve(b1))


@pytest.mark.parametrize("cycle", ["V", "W", "F"])
@pytest.mark.parametrize("gi", list(GEOMS))
def test_polar_mg_cycle_bitexact(problems, gi, cycle):
    d, o = problems[gi]
    L = d.num_levels
    u0 = Oracle.random_vector(d.n(L), 3)
    g = Oracle.random_vector(d.n(L), 4)
    for steps in ((2, 2), (3, 1), (1, 5)):
        spec = dict(cycle=cycle, smoother="jacobi", pre_steps=steps[0], post_steps=steps[1])
        got = gmg.mg_cycle(d, L, u0, g, gmg.CycleSpec(**spec))
        want = o.mg_cycle(OSpec(**spec), L, u0, g)
        assert bits_equal(got, want), (cycle, steps, first_mismatch(got, want))


@pytest.mark.parametrize("gi", list(GEOMS))
def test_polar_solve_bitexact(problems, gi):
    d, o = problems[gi]
    L = d.num_levels
    n = d.n(L)
    b = Oracle.random_vector(n, 1)
    for kw in (dict(tolerance=1e-8, max_cycles=25), dict(tolerance=1e-9, max_cycles=15, adaptive_correction=False,
                                                           correction_omega=2.0)):
        spec = dict(smoother="jacobi", smoothing_omega=0.7, **kw)
        xg, xo = np.zeros(n), np.zeros(n)
        rg = gmg.solve(d, b, gmg.CycleSpec(**spec), xg)
        ro = o.solve(OSpec(**spec), b, xo)
        assert rg.iterations == ro.iterations
        assert bits_equal(np.asarray(rg.residual_history), np.asarray(ro.history))
        assert bits_equal(xg, xo), first_mismatch(xg, xo)


def test_polar_nested_start_vector(problems):
    d, o = problems["L5_c2"]
    b = Oracle.random_vector(d.n(5), 9)
    spec = dict(smoother="jacobi", smoothing_omega=0.7)
    assert bits_equal(gmg.make_start_vector("nested", d, gmg.CycleSpec(**spec), b), o.start_vector(OSpec(**spec), "nested", b))


def test_polar_rejects_sweeps_and_slabs(problems):
    d, _ = problems["L5_c2"]
    n = d.n(5)
    with pytest.raises(gmg.InvalidArgument, match="periodic"):
        gmg.solve(d, np.ones(n), gmg.CycleSpec(smoother="gauss_seidel"), np.zeros(n))
    with pytest.raises(gmg.InvalidArgument, match="periodic"):
        gmg.MultilevelProblem(5, 1, 2, (1.0, 1.0), "polar", 1.0, 1.0, slabs=gmg.Slabs(world=2, min_rows=4))


@pytest.mark.slow
def test_c3_polar_full_size(gpu):
    """BASELINE configs[2]: 1023 x 1024 (r x theta; 1025^2 vertices with the periodic seam),
    10 levels, seeded U[-1,1] f, zero start, F-cycle, jacobi 0.7 2+2, adaptive omega_l,
    stop at 1e-8 (capped at the reference default of 50 cycles)."""
    a = (10, 1, 2, (1.0, 1.0), "polar", 1.0, 1.0)
    d, o = gmg.MultilevelProblem(*a), Oracle(*a)
    assert d.shapes[10] == (1023, 1024)
    n = d.n(10)
    b = Oracle.random_vector(n, 1)
    spec = dict(smoother="jacobi", smoothing_omega=0.7, pre_steps=2, post_steps=2, tolerance=1e-8, max_cycles=50)
    xg, xo = np.zeros(n), np.zeros(n)
    rg = gmg.solve(d, b, gmg.CycleSpec(**spec), xg)
    ro = o.solve(OSpec(**spec), b, xo)
    assert rg.iterations == ro.iterations
    assert bits_equal(np.asarray(rg.residual_history), np.asarray(ro.history)), \
        first_mismatch(rg.residual_history, ro.history)
    assert bits_equal(xg, xo), first_mismatch(xg, xo)
