"""Row-slab distribution on one GPU: every slab of
a `world`-rank group runs in this process on the same device and stream
(virtual ranks), exchanging halo rows, threshold gathers and the exact-sum
state handoff by device copies — the same schedule the NCCL transport runs
across processes. The result must be bit-identical to the single-domain solve
(and therefore to the reference): sharding does not change any per-element
arithmetic, and the reductions are chained in rank order.
"""
import numpy as np
import pytest

from conftest import bits_equal, first_mismatch

gmg = pytest.importorskip("paper_0805_3041_b200.gmg")

pytestmark = pytest.mark.gpu


def solve_pair(args, spec, world, min_rows, seed_x=0):
    single = gmg.MultilevelProblem(*args)
    slab = gmg.MultilevelProblem(*args, slabs=gmg.Slabs(world=world, min_rows=min_rows))
    L = single.num_levels
    n = single.n(L)
    b = gmg.random_vector(n, 1)
    x0 = gmg.random_vector(n, seed_x) if seed_x else np.zeros(n)
    xs, xd = x0.copy(), x0.copy()
    rs = gmg.solve(single, b, spec, xs)
    rd = gmg.solve(slab, b, spec, xd)
    return single, slab, rs, rd, xs, xd


@pytest.mark.parametrize("world", [2, 3, 4])
@pytest.mark.parametrize("cycle", ["F", "V", "W"])
def test_slab_solve_bitexact(gpu, world, cycle):
    args = (7, 1, 1, (1.0, 1.0), "cartesian", 1.0, 1.0)
    spec = gmg.CycleSpec(cycle=cycle, smoother="jacobi", tolerance=1e-10, max_cycles=30)
    single, slab, rs, rd, xs, xd = solve_pair(args, spec, world, min_rows=15)
    rank, w, Ls = slab.dist_info()
    assert (rank, w) == (0, world) and Ls <= 5  # levels >= Ls are really split
    assert rs.iterations == rd.iterations
    assert bits_equal(np.array(rs.residual_history), np.array(rd.residual_history))
    assert bits_equal(xs, xd), first_mismatch(xs, xd)


@pytest.mark.parametrize("pre,post", [(2, 2), (1, 3), (0, 2), (5, 6)])
def test_slab_steps_and_fixed_omega(gpu, pre, post):
    # steps > 4 need several fused launches with a halo refresh between them
    args = (7, 2, 1, (1.0, 1.0), "cartesian", 0.3, 1.0)
    for adaptive in (True, False):
        spec = gmg.CycleSpec(smoother="jacobi", pre_steps=pre, post_steps=post, adaptive_correction=adaptive,
                             correction_omega=1.5, tolerance=1e-9, max_cycles=20)
        _, _, rs, rd, xs, xd = solve_pair(args, spec, 3, min_rows=15, seed_x=2)
        assert rs.residual_history == rd.residual_history, (pre, post, adaptive)
        assert bits_equal(xs, xd)


@pytest.mark.parametrize("coords", ["cylindrical", "spherical"])
def test_slab_non_constant_operators(gpu, coords):
    args = (6, 2, 3, (1.05, 0.97), coords, 1.0, 0.5)
    spec = gmg.CycleSpec(smoother="jacobi", tolerance=1e-9, max_cycles=25)
    _, _, rs, rd, xs, xd = solve_pair(args, spec, 2, min_rows=20)
    assert rs.residual_history == rd.residual_history
    assert bits_equal(xs, xd)


@pytest.mark.parametrize("world", [2, 8])
def test_slab_large_levels_engine_path(gpu, world):
    # 1023^2: per-slab sums far above the direct-kernel size, so the walk/chain
    # engine runs per slab and chains across slabs
    args = (10, 1, 1, (1.0, 1.0), "cartesian", 1.0, 1.0)
    spec = gmg.CycleSpec(smoother="jacobi", tolerance=1e-10, max_cycles=12)
    single, slab, rs, rd, xs, xd = solve_pair(args, spec, world, min_rows=255)
    assert slab.dist_info()[2] == 8
    assert rs.iterations == rd.iterations and rs.residual_history == rd.residual_history
    assert bits_equal(xs, xd)


def test_slab_fast_reduction_close(gpu):
    args = (8, 1, 1, (1.0, 1.0), "cartesian", 1.0, 1.0)
    spec = gmg.CycleSpec(smoother="jacobi", tolerance=1e-9, max_cycles=15, reduction="fast")
    _, _, rs, rd, xs, xd = solve_pair(args, spec, 4, min_rows=31)
    assert rs.iterations == rd.iterations
    np.testing.assert_allclose(rd.residual_history, rs.residual_history, rtol=1e-6)


def test_slab_handle_rejects_unsharded_ops(gpu):
    slab = gmg.MultilevelProblem(6, slabs=gmg.Slabs(world=2, min_rows=15))
    n = slab.n(6)
    with pytest.raises(gmg.LogicError, match="row-slab handle"):
        gmg.apply(slab, 6, np.zeros(n))
    with pytest.raises(gmg.Unsupported, match="jacobi"):
        gmg.solve(slab, np.ones(n), gmg.CycleSpec(smoother="gauss_seidel"), np.zeros(n))


def test_nccl_group_of_one(gpu):
    # the multi-process entry point end to end on one GPU: NCCL loaded and a
    # one-rank communicator created (nothing is sharded with one rank)
    uid = gmg.unique_id()
    assert len(uid) == 128
    args = (7, 1, 1, (1.0, 1.0), "cartesian", 1.0, 1.0)
    p1 = gmg.MultilevelProblem(*args, slabs=gmg.Slabs(world=1, rank=0, min_rows=15, nccl_id=uid))
    assert p1.dist_info() == (0, 1, 8)
    single = gmg.MultilevelProblem(*args)
    n = single.n(7)
    b = gmg.random_vector(n, 1)
    spec = gmg.CycleSpec(smoother="jacobi", tolerance=1e-10)
    x1, x2 = np.zeros(n), np.zeros(n)
    r1, r2 = gmg.solve(p1, b, spec, x1), gmg.solve(single, b, spec, x2)
    assert r1.residual_history == r2.residual_history and bits_equal(x1, x2)
