"""Parity of the non-Jacobi smoothers on the device:
richardson, ilu0 and the line smoothers tri_x, tri_y, adi, gstri_x, gstri_y,
gsadi (reference smoother.cpp:74-386), against the reference's golden
smooth_step vectors and against the oracle at every level, in mg_cycle and
in whole solves. Bit-for-bit throughout.
"""
import numpy as np
import pytest

from conftest import bits_equal, first_mismatch, load_golden, unhex
from pyoracle import CycleSpec as OSpec
from pyoracle import Oracle

gmg = pytest.importorskip("paper_0805_3041_b200.gmg")

pytestmark = pytest.mark.gpu

NEW_KINDS = ["richardson", "ilu0", "tri_x", "tri_y", "adi", "gstri_x", "gstri_y", "gsadi"]
LINE_KINDS = ["tri_x", "tri_y", "adi", "gstri_x", "gstri_y", "gsadi"]
OPS_FIXTURES = ["ops_cartesian_uniform", "ops_cartesian_aniso", "ops_cylindrical", "ops_spherical_graded"]

GEOMS = {
    "cart": dict(levels=5, coarse=(1, 1), coords="cartesian", alpha=1.0, beta=1.0, grading=(1.0, 1.0)),
    "aniso_rect": dict(levels=4, coarse=(2, 3), coords="cartesian", alpha=1e-2, beta=1.0, grading=(1.0, 1.0)),
    "cyl": dict(levels=5, coarse=(1, 1), coords="cylindrical", alpha=1.0, beta=1.0, grading=(1.0, 1.0)),
    "sph": dict(levels=4, coarse=(3, 2), coords="spherical", alpha=1.3, beta=0.7, grading=(1.1, 0.93)),
    "wide": dict(levels=3, coarse=(60, 1), coords="cartesian", alpha=0.5, beta=2.0, grading=(1.0, 1.02)),
    # 255 x 383: several wavefront CTAs, partial line blocks, lines longer than a chunk
    "tall": dict(levels=7, coarse=(1, 2), coords="cartesian", alpha=0.3, beta=1.0, grading=(1.0, 1.0)),
    # wavefront edge cases: widths that are no multiple of the 16-column staging block (the reversed
    # ILU wave shifts its clock), a last warp with a single row (33 rows), fewer columns than a window
    "odd_39x15": dict(levels=4, coarse=(4, 1), coords="cartesian", alpha=0.7, beta=1.0, grading=(1.0, 1.0)),
    "odd_47x39": dict(levels=3, coarse=(11, 9), coords="cartesian", alpha=1e-3, beta=1.0, grading=(1.0, 1.0)),
    "odd_41x33": dict(levels=2, coarse=(20, 16), coords="cylindrical", alpha=1.0, beta=1.0, grading=(1.0, 1.0)),
    "odd_9x65": dict(levels=2, coarse=(4, 32), coords="cartesian", alpha=1.0, beta=1.0, grading=(1.03, 1.0)),
}


def args(geom):
    return (geom["levels"], geom["coarse"][0], geom["coarse"][1], geom["grading"], geom["coords"],
            geom["alpha"], geom["beta"])


@pytest.fixture(scope="module")
def problems(gpu):
    return {k: (gmg.MultilevelProblem(*args(g)), Oracle(*args(g))) for k, g in GEOMS.items()}


@pytest.mark.parametrize("name", OPS_FIXTURES)
def test_smooth_step_matches_reference_golden(gpu, name):
    g = load_golden(name)
    pb = g["problem"]
    d = gmg.MultilevelProblem(pb["levels"], pb["coarse_nx"], pb["coarse_ny"], tuple(pb["grading"]), pb["coords"],
                              pb["alpha"], pb["beta"])
    for ls, e in g["levels"].items():
        l = int(ls)
        x = gmg.random_vector(d.n(l), e["x_seed"])
        b = gmg.random_vector(d.n(l), e["b_seed"])
        for k, s in e["smooth_step"].items():
            got = gmg.smooth_step(d, l, k, s["smoother_omega"], x, b, s["omega_damp"])
            want = unhex(s["out"])
            assert bits_equal(got, want), (name, l, k, first_mismatch(got, want))


@pytest.mark.parametrize("gi", list(GEOMS))
def test_smooth_step_all_kinds_every_level(problems, gi):
    d, o = problems[gi]
    for l in range(1, d.num_levels + 1):
        n = d.n(l)
        x = Oracle.random_vector(n, 60 + l)
        b = Oracle.random_vector(n, 70 + l)
        cases = [("richardson", 1.0), ("richardson", 1e-4), ("ilu0", 1.0), ("ilu0", 0.5),
                 ("gauss_seidel", 1.0), ("sor", 1.3), ("sor", 0.4)]
        cases += [(k, w) for k in LINE_KINDS for w in (1.0, 0.6)]
        for kind, som in cases:
            for damp in (0.7, 1.0):
                got = gmg.smooth_step(d, l, kind, som, x, b, damp)
                want = o.smooth_step(l, kind, som, damp, x, b)
                assert bits_equal(got, want), (gi, l, kind, som, damp, first_mismatch(got, want))


@pytest.mark.parametrize("kind", NEW_KINDS)
@pytest.mark.parametrize("cycle", ["V", "W"])
def test_mg_cycle_new_smoothers(problems, kind, cycle):
    for gi in ("cart", "sph"):
        d, o = problems[gi]
        spec = dict(cycle=cycle, smoother=kind, smoother_omega=0.9 if kind in LINE_KINDS else 1.0, pre_steps=1,
                    post_steps=2, adaptive_correction=True)
        for l in range(1, d.num_levels + 1):
            u0 = Oracle.random_vector(d.n(l), 80 + l)
            g = Oracle.random_vector(d.n(l), 90 + l)
            got = gmg.mg_cycle(d, l, u0, g, gmg.CycleSpec(**spec))
            want = o.mg_cycle(OSpec(**spec), l, u0, g)
            assert bits_equal(got, want), (gi, cycle, kind, l, first_mismatch(got, want))


@pytest.mark.parametrize("kind", NEW_KINDS)
@pytest.mark.parametrize("gi", ["cart", "cyl", "aniso_rect"])
def test_solve_new_smoothers_bitexact(problems, kind, gi):
    d, o = problems[gi]
    L = d.num_levels
    n = d.n(L)
    b = Oracle.random_vector(n, 1)
    x0 = Oracle.random_vector(n, 2)
    kw = dict(cycle="F", smoother=kind, smoother_omega=1.0, pre_steps=2, post_steps=2, tolerance=1e-10,
              max_cycles=12)
    xg = x0.copy()
    xo = x0.copy()
    try:
        rg = gmg.solve(d, b, gmg.CycleSpec(**kw), xg)
        hist = rg.residual_history
    except gmg.DivergenceError as e:
        hist = e.report.residual_history
    ro = o.solve(OSpec(**kw), b, xo)
    assert len(hist) == len(ro.history) and bits_equal(np.asarray(hist), np.asarray(ro.history)), (kind, gi)
    assert bits_equal(xg, xo), (kind, gi, first_mismatch(xg, xo))


def test_richardson_clamp_matches_oracle(problems):
    # omega above 1/lambda_max is clamped to 0.9/lambda_max at setup (smoother.cpp:243-247)
    d, o = problems["cart"]
    l = d.num_levels
    x = Oracle.random_vector(d.n(l), 3)
    b = Oracle.random_vector(d.n(l), 4)
    for som in (0.5, 5.0, 1e3):
        got = gmg.smooth_step(d, l, "richardson", som, x, b, 1.0)
        want = o.smooth_step(l, "richardson", som, 1.0, x, b)
        assert bits_equal(got, want), som


def test_line_smoother_omega_range_is_checked(problems):
    d, _ = problems["cart"]
    n = d.n(d.num_levels)
    for kind in LINE_KINDS:
        with pytest.raises(gmg.InvalidArgument, match=r"\(0, 1\] for line smoothers"):
            gmg.solve(d, np.ones(n), gmg.CycleSpec(smoother=kind, smoother_omega=1.5), np.zeros(n))
    with pytest.raises(gmg.InvalidArgument, match="must be > 0"):
        gmg.solve(d, np.ones(n), gmg.CycleSpec(smoother="ilu0", smoother_omega=0.0), np.zeros(n))


@pytest.mark.slow
@pytest.mark.parametrize("kind", ["adi", "gsadi", "ilu0"])
def test_solve_1023_line_and_ilu_bitexact(gpu, kind):
    """C2/C3'-size grids (1023^2, 10 levels): whole-grid wavefront (ilu0) and per-line
    (adi) / serial-chain (gsadi) kernels at full size, 3 F-cycles from a random start,
    anisotropic eps = 1e-2 (the paper's line-smoother case): histories and solution
    bit for bit against the oracle."""
    a = (10, 1, 1, (1.0, 1.0), "cartesian", 1e-2, 1.0)
    d, o = gmg.MultilevelProblem(*a), Oracle(*a)
    n = d.n(10)
    b = Oracle.random_vector(n, 1)
    x0 = Oracle.random_vector(n, 2)
    kw = dict(cycle="F", smoother=kind, smoother_omega=1.0 if kind != "ilu0" else 1.1, pre_steps=2,
              post_steps=2, tolerance=1e-30, max_cycles=3)
    xg, xo = x0.copy(), x0.copy()
    rg = gmg.solve(d, b, gmg.CycleSpec(**kw), xg)
    ro = o.solve(OSpec(**kw), b, xo)
    assert rg.iterations == ro.iterations == 3
    assert bits_equal(np.asarray(rg.residual_history), np.asarray(ro.history)), kind
    assert bits_equal(xg, xo), (kind, first_mismatch(xg, xo))
