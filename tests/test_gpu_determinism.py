"""Run-to-run determinism of the kernels whose CTAs cooperate through global
memory (compute-sanitizer's racecheck/synccheck are closed on this pool, see
DESIGN.md §4): the Gauss-Seidel and ILU(0) wavefronts (warp-edge rows and
progress counters shared between CTAs, gs.cuh) and the exact-sum engine's
decoupled look-backs (seqsum.cuh). A missed dependency would show up as a
result that changes between repetitions or departs from the sequential oracle;
both are checked bit for bit over repeated runs."""
import numpy as np
import pytest

from conftest import bits_equal
from pyoracle import CycleSpec as OSpec
from pyoracle import Oracle

gmg = pytest.importorskip("paper_0805_3041_b200.gmg")

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("kind,levels", [("gauss_seidel", 10), ("sor", 9), ("ilu0", 9)])
def test_wavefront_solves_repeat_bitexact(gpu, kind, levels):
    a = (levels, 1, 1, (1.0, 1.0), "cartesian", 1e-2, 1.0)
    d = gmg.MultilevelProblem(*a)
    n = d.n(levels)
    b = gmg.random_vector(n, 1)
    x0 = gmg.random_vector(n, 2)
    spec = gmg.CycleSpec(smoother=kind, smoother_omega=1.2 if kind == "sor" else 1.0, tolerance=1e-30, max_cycles=2)
    ref_x, ref_h = None, None
    for _ in range(5):
        x = x0.copy()
        r = gmg.solve(d, b, spec, x)
        if ref_x is None:
            ref_x, ref_h = x, r.residual_history
        assert r.residual_history == ref_h and bits_equal(x, ref_x)
    o = Oracle(*a)
    xo = x0.copy()
    ro = o.solve(OSpec(smoother=kind, smoother_omega=1.2 if kind == "sor" else 1.0, tolerance=1e-30, max_cycles=2), b, xo)
    assert bits_equal(np.asarray(ref_h), np.asarray(ro.history)) and bits_equal(ref_x, xo)


def test_exact_sums_repeat_bitexact(gpu):
    d = gmg.MultilevelProblem(12)  # the workspace of a 4095^2 finest level
    rng = np.random.default_rng(5)
    for n in (4097, 1 << 16, (1 << 20) + 7, 1 << 23):
        v = rng.standard_normal(n) * np.exp2(rng.integers(-30, 30, n))
        w = rng.standard_normal(n)
        want_n = Oracle.load().orc_norm_l2(n, v.ctypes.data_as(__import__("ctypes").POINTER(__import__("ctypes").c_double)))
        want_d = Oracle(1).dot(v, w)
        for _ in range(4):
            assert gmg.norm_l2(d, v) == want_n
            assert gmg.dot(d, v, w) == want_d
