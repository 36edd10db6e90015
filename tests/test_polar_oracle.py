"""The polar-periodic restatement (BASELINE config 3, no reference counterpart:
parity unpinned) checked on the CPU through properties that do
not need a reference: the operator is symmetric, theta-periodic, and the whole
multigrid cycle commutes with a rotation by a multiple of the coarsest theta
spacing (every level's node set maps onto itself), bit for bit with a fixed
correction weight. CPU only (oracle/gmg_oracle.c)."""
import numpy as np
import pytest

from conftest import bits_equal
from pyoracle import CheckerError, CycleSpec, Oracle


def polar(levels, cny=2, cnx=1, gx=1.0, alpha=1.0, beta=1.0):
    return Oracle(levels, cnx, cny, (gx, 1.0), "polar", alpha, beta)


def roll_rows(v, nx, ny, k):
    return np.roll(v.reshape(ny, nx), k, axis=0).ravel()


def test_polar_hierarchy_shapes():
    o = polar(5, cny=2, cnx=1)
    assert [(o.shapes[l]) for l in range(1, 6)] == [(1, 2), (3, 4), (7, 8), (15, 16), (31, 32)]
    x, y = o.coords(5)
    assert x[0] == 0.1 and x[-1] == 1.0
    assert np.array_equal(y, np.arange(34) / 32.0)  # dyadic theta/(2 pi) nodes incl. the wrapped neighbours


def test_polar_operator_symmetric_and_periodic():
    o = polar(4, cny=4, gx=1.05)
    L = 4
    nx, ny = o.shapes[L]
    op = o.operator(L)
    # coefficients depend on r only, s/n couple across the wrap
    C = op["c"].reshape(ny, nx)
    assert np.all(C == C[0]) and np.all(op["s"] != 0) and np.all(op["n"] != 0)
    a = Oracle.random_vector(nx * ny, 1)
    b = Oracle.random_vector(nx * ny, 2)
    assert abs(a @ o.apply(L, b) - b @ o.apply(L, a)) < 1e-12 * np.abs(a).sum()
    # theta rotation by one row commutes with A exactly (the stencil is row-invariant)
    assert bits_equal(o.apply(L, roll_rows(a, nx, ny, 1)), roll_rows(o.apply(L, a), nx, ny, 1))


@pytest.mark.parametrize("cycle", ["V", "W", "F"])
def test_polar_cycle_commutes_with_rotation(cycle):
    L = 5
    o = polar(L, cny=2, alpha=0.7)
    nx, ny = o.shapes[L]
    shift = ny // 2  # one coarsest theta spacing (level 1 has 2 nodes)
    g = Oracle.random_vector(nx * ny, 3)
    u0 = Oracle.random_vector(nx * ny, 4)
    # level 1 smoothed instead of factored: a Cholesky solve is not permutation-equivariant
    # in its rounding, Jacobi sweeps are
    spec = CycleSpec(cycle=cycle, smoother="jacobi", adaptive_correction=False, correction_omega=1.7,
                     coarse_direct_max_neq=0)
    u = o.mg_cycle(spec, L, u0, g)
    ur = o.mg_cycle(spec, L, roll_rows(u0, nx, ny, shift), roll_rows(g, nx, ny, shift))
    assert bits_equal(ur, roll_rows(u, nx, ny, shift))


def test_polar_solve_converges_and_rejects_sweeps():
    o = polar(6, cny=2)
    n = o.n(6)
    b = Oracle.random_vector(n, 1)
    r = o.solve(CycleSpec(smoother="jacobi", smoothing_omega=0.7, tolerance=1e-8, max_cycles=200), b, np.zeros(n))
    assert r.status == 0 and r.history[-1] < r.history[0] * 1e-3
    r = o.solve(CycleSpec(smoother="gauss_seidel"), b, np.zeros(n))
    assert r.status == 2 and "periodic" in r.message
    with pytest.raises(CheckerError, match="uniform"):
        Oracle(3, 1, 2, (1.0, 1.1), "polar", 1.0, 1.0)
