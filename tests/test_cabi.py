"""CPU-side checks of the C-ABI library (no device compute):
the .so loads, exports every symbol include/gmg_b200.h declares, its host
helpers are exact (seeded input generator; the exact-order summation engine's
logic via its host emulation), and host-side validation raises the reference's
exception types before any device work."""
import ctypes
import os
import re

import numpy as np
import pytest

from conftest import ROOT, bits_equal, has_gpu, load_golden, unhex

gmg = pytest.importorskip("paper_0805_3041_b200.gmg")


def declared_symbols():
    text = open(os.path.join(ROOT, "include", "gmg_b200.h")).read()
    return sorted(set(re.findall(r"\b(gmg_(?:dev|host|dist)_\w+|gmg_last_error|gmg_version)\s*\(", text)))


def test_library_exports_every_declared_symbol():
    lib = gmg.lib()
    syms = declared_symbols()
    assert len(syms) >= 20
    missing = [s for s in syms if not hasattr(lib, s)]
    assert not missing, missing
    assert sorted(gmg.EXPORTS) == syms


def test_library_is_sm100a():
    lib = gmg.lib()
    assert b"sm_100a" in lib.gmg_version()


def test_random_vector_is_the_reference_generator():
    g = load_golden("random_vector")
    assert bits_equal(gmg.random_vector(g["n"], g["seed"]), unhex(g["values"]))


def _seq(t):
    s = 0.0
    for v in t:
        s += v
    return s


def _cases():
    rng = np.random.default_rng(11)
    yield "empty", np.zeros(0)
    yield "single", np.array([3.25])
    yield "mixed", rng.uniform(-1, 1, 70001)
    yield "positive", rng.uniform(0, 1, 50000) ** 2
    yield "dyadic_ties", np.ldexp(np.round(rng.uniform(-8, 8, 40000)), -rng.integers(0, 4, 40000))
    yield "magnitudes", rng.uniform(-1, 1, 30000) * 10.0 ** rng.integers(-15, 15, 30000)
    yield "cancellation", np.where(rng.random(60000) < 0.5, -1.0, 1.0) * (1 + 1e-9 * rng.uniform(-1, 1, 60000))
    v = rng.uniform(-1, 1, 20000) * 1e-300
    v[::997] = 1e300
    yield "extremes", v
    yield "zeros_then_values", np.concatenate([np.zeros(9000), rng.uniform(-1, 1, 9000)])
    yield "exact_cancel", np.tile([1.0, -1.0, 2.0 ** -60], 12000)


@pytest.mark.parametrize("name,terms", list(_cases()), ids=[c[0] for c in _cases()])
def test_exact_sum_engine_logic_matches_sequential(name, terms):
    got, stats = gmg.seqsum_emulate(terms)
    want = _seq(terms.tolist())
    assert bits_equal(np.array([got]), np.array([want])), (got, want, stats)


@pytest.mark.parametrize("threads,ept", [(256, 32), (32, 4), (7, 3), (1, 1)])
def test_exact_sum_engine_any_chunking(threads, ept):
    rng = np.random.default_rng(threads * 31 + ept)
    terms = rng.uniform(-1, 1, 12345) * rng.uniform(0, 1, 12345)
    got, _ = gmg.seqsum_emulate(terms, threads, ept)
    assert got == _seq(terms.tolist())


def test_host_validation_precedes_device_work():
    with pytest.raises(gmg.InvalidArgument, match="levels"):
        gmg.MultilevelProblem(0)
    with pytest.raises(gmg.InvalidArgument, match="alpha/beta"):
        gmg.MultilevelProblem(3, alpha=0.0)
    with pytest.raises(gmg.InvalidArgument, match="coarse_n"):
        gmg.MultilevelProblem(3, coarse_nx=0)
    with pytest.raises(gmg.InvalidArgument, match="grading"):
        gmg.MultilevelProblem(3, grading=(-1.0, 1.0))
    with pytest.raises(gmg.InvalidArgument):
        gmg.CycleSpec(cycle="X")._c()


@pytest.mark.skipif(has_gpu(), reason="checks the no-GPU failure mode")
def test_no_device_fails_loudly():
    with pytest.raises(gmg.CudaError):
        gmg.MultilevelProblem(3)
