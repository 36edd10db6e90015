"""Study-layer callers on the device: make_start_vector
(study.cpp:40-79) through gmg_dev_make_start_vector, bit for bit against the
oracle restatement (which test_oracle_pin.py pins to the reference's own
make_start_vector). The full run_study sweep on the GPU backend is compared
with the reference's run_study in oracle/shim_demo.cpp (test_integration.py).
"""
import numpy as np
import pytest

from conftest import bits_equal, first_mismatch
from pyoracle import CycleSpec as OSpec
from pyoracle import Oracle

gmg = pytest.importorskip("paper_0805_3041_b200.gmg")

pytestmark = pytest.mark.gpu

CASES = [
    # levels, coarse, coords, alpha, grading, smoother, smoother_omega
    (7, (1, 1), "cartesian", 1.0, (1.0, 1.0), "jacobi", 1.0),
    (9, (1, 1), "cartesian", 1e-2, (1.0, 1.0), "jacobi", 1.0),  # 511^2: warp-strip kernels
    (6, (2, 3), "cylindrical", 0.3, (1.0, 1.0), "gauss_seidel", 1.0),
    (5, (1, 1), "spherical", 1.3, (1.1, 0.93), "adi", 0.9),
    (5, (3, 2), "cartesian", 0.1, (1.0, 1.02), "ilu0", 1.1),
    (5, (1, 1), "cartesian", 1.0, (1.0, 1.0), "richardson", 5.0),
    (5, (1, 1), "cylindrical", 1.0, (1.0, 1.0), "gsadi", 1.0),
    (1, (5, 4), "cartesian", 1.0, (1.0, 1.0), "sor", 1.3),  # single level: the direct solve
]


@pytest.mark.parametrize("case", CASES, ids=[f"{c[5]}-{c[2]}-L{c[0]}" for c in CASES])
@pytest.mark.parametrize("kind", ["zero", "nested"])
def test_make_start_vector_bitexact(gpu, case, kind):
    levels, coarse, coords, alpha, grading, sm, som = case
    a = (levels, coarse[0], coarse[1], grading, coords, alpha, 1.0)
    d, o = gmg.MultilevelProblem(*a), Oracle(*a)
    b = Oracle.random_vector(d.n(levels), 5)
    spec = dict(smoother=sm, smoother_omega=som, smoothing_omega=0.7)
    got = gmg.make_start_vector(kind, d, gmg.CycleSpec(**spec), b)
    want = o.start_vector(OSpec(**spec), kind, b)
    assert bits_equal(got, want), first_mismatch(got, want)


def test_nested_start_then_solve(gpu):
    """run_one's order (study.cpp:169-177): b, nested start vector, solve — all on the device."""
    a = (8, 1, 1, (1.0, 1.0), "cartesian", 0.1, 1.0)
    d, o = gmg.MultilevelProblem(*a), Oracle(*a)
    n = d.n(8)
    b = Oracle.random_vector(n, 1)
    kw = dict(smoother="gauss_seidel", smoothing_omega=0.7, tolerance=1e-8)
    xg = gmg.make_start_vector("nested", d, gmg.CycleSpec(**kw), b)
    xo = o.start_vector(OSpec(**kw), "nested", b)
    rg = gmg.solve(d, b, gmg.CycleSpec(**kw), xg)
    ro = o.solve(OSpec(**kw), b, xo)
    assert rg.iterations == ro.iterations
    assert bits_equal(np.asarray(rg.residual_history), np.asarray(ro.history))
    assert bits_equal(xg, xo)


def test_start_vector_errors(gpu):
    d = gmg.MultilevelProblem(4)
    n = d.n(4)
    with pytest.raises(gmg.InvalidArgument, match="continuation requires a source"):
        gmg.make_start_vector("continuation", d, gmg.CycleSpec(), np.ones(n))
    with pytest.raises(gmg.InvalidArgument, match="shape does not match"):
        gmg.make_start_vector("continuation", d, gmg.CycleSpec(), np.ones(n), source=np.ones(n + 1))
    src = np.arange(n, dtype=np.float64)
    assert np.array_equal(gmg.make_start_vector("continuation", d, gmg.CycleSpec(), np.ones(n), source=src), src)
    with pytest.raises(gmg.InvalidArgument, match="must be in \\(0, 2\\)"):
        gmg.make_start_vector("nested", d, gmg.CycleSpec(smoother="sor", smoother_omega=2.5), np.ones(n))


def test_make_start_vector_matches_reference_golden(gpu):
    from conftest import load_golden, unhex
    g = load_golden("start_vectors")
    for case in g["cases"]:
        pb = case["problem"]
        d = gmg.MultilevelProblem(pb["levels"], pb["coarse_nx"], pb["coarse_ny"], tuple(pb["grading"]),
                                  pb["coords"], pb["alpha"], pb["beta"])
        b = gmg.random_vector(d.n(pb["levels"]), case["b_seed"])
        got = gmg.make_start_vector("nested", d, gmg.CycleSpec(**case["spec"]), b)
        assert bits_equal(got, unhex(case["nested"])), (case["spec"]["smoother"], first_mismatch(got, unhex(case["nested"])))
