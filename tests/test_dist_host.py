"""Host side of the row-slab multi-GPU path, on CPU with two
`gloo` processes: the partition every rank computes (gmg_host_slab_plan in
libgmg_b200.so), the halo schedule of dist_halo, the threshold gather and the
rank-ordered exact-sum handoff, replayed with torch.distributed point-to-point
messages over numpy slabs and checked bit for bit against the single-domain
oracle. No GPU: the CUDA kernels' share of the same schedule is covered by
tests/test_gpu_slabs.py (virtual ranks on one device).
"""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from pyoracle import Oracle

gmg = pytest.importorskip("paper_0805_3041_b200.gmg")

H = 4  # halo rows (DistCtx::H)


def free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _exchange_halo(buf, w0, w1, rank, world, rows):
    """dist_halo: my first rows -> rank-1, my last rows -> rank+1 (and the converse)."""
    nx = buf.shape[1]
    reqs = []
    recv_up = recv_dn = None
    if rank > 0:
        reqs.append(dist.isend(torch.from_numpy(np.ascontiguousarray(buf[w0:w0 + rows])), rank - 1))
        recv_up = torch.empty((rows, nx), dtype=torch.float64)
        reqs.append(dist.irecv(recv_up, rank - 1))
    if rank + 1 < world:
        reqs.append(dist.isend(torch.from_numpy(np.ascontiguousarray(buf[w1 - rows:w1])), rank + 1))
        recv_dn = torch.empty((rows, nx), dtype=torch.float64)
        reqs.append(dist.irecv(recv_dn, rank + 1))
    for r in reqs:
        r.wait()
    if recv_up is not None:
        buf[w0 - rows:w0] = recv_up.numpy()
    if recv_dn is not None:
        buf[w1:w1 + rows] = recv_dn.numpy()


def _worker(rank, world, port, out):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        args = (7, 1, 1, (1.0, 1.0), "cartesian", 0.5, 1.0)
        o = Oracle(*args)
        L = 7
        ny = [o.shapes[l][1] for l in range(1, L + 1)]
        Ls, W0, W1 = gmg.slab_plan(ny, world, min_rows=15, halo=H)
        # 1. every rank derives the same plan
        plans = [None] * world
        dist.all_gather_object(plans, (Ls, W0, W1))
        assert all(p == plans[0] for p in plans)
        # 2. windows tile every level; sharded levels nest by factor two; >= H rows each
        for l in range(1, L + 1):
            w0, w1 = W0[l - 1], W1[l - 1]
            if l < Ls:
                assert w0 == [0] * world and w1 == [ny[l - 1]] * world
                continue
            assert w0[0] == 0 and w1[-1] == ny[l - 1]
            assert all(w1[r] == w0[r + 1] for r in range(world - 1))
            assert all(w1[r] - w0[r] >= H for r in range(world))
            if l > Ls:
                assert all(w0[r] == 2 * W0[l - 2][r] for r in range(1, world))
        # 3. a Jacobi smooth_step on every sharded level from owned rows + exchanged halo
        #    equals the single-domain step on the owned rows
        for l in range(Ls, L + 1):
            nx, nyl = o.shapes[l]
            x = Oracle.random_vector(nx * nyl, 10 + l).reshape(nyl, nx)
            b = Oracle.random_vector(nx * nyl, 20 + l).reshape(nyl, nx)
            full = o.smooth_step(l, "jacobi", 1.0, 0.7, x.ravel(), b.ravel()).reshape(nyl, nx)
            w0, w1 = W0[l - 1][rank], W1[l - 1][rank]
            mine = np.full_like(x, np.nan)
            mine[w0:w1] = x[w0:w1]
            _exchange_halo(mine, w0, w1, rank, world, H)
            lo, hi = max(0, w0 - 1), min(nyl, w1 + 1)
            assert not np.isnan(mine[lo:hi]).any()
            local = np.where(np.isnan(mine), 0.0, mine)  # rows beyond the halo never reach owned rows
            got = o.smooth_step(l, "jacobi", 1.0, 0.7, local.ravel(), b.ravel()).reshape(nyl, nx)
            assert np.array_equal(got[w0:w1].view(np.uint64), full[w0:w1].view(np.uint64)), l
        # 4. threshold gather: the coarse rows each rank restricts into tile level Ls-1
        if Ls > 1:
            a = [W0[Ls - 1][r] // 2 for r in range(world)]
            bnd = [W1[Ls - 1][r] // 2 for r in range(world)]
            assert a[0] == 0 and bnd[-1] == ny[Ls - 2] and all(bnd[r] == a[r + 1] for r in range(world - 1))
        # 5. exact-sum handoff: each rank continues the left-to-right sum from its
        #    predecessor's exact state; the last rank holds the reference's sum
        nx, nyl = o.shapes[L]
        t = Oracle.random_vector(nx * nyl, 5).reshape(nyl, nx) * Oracle.random_vector(nx * nyl, 6).reshape(nyl, nx)
        w0, w1 = W0[L - 1][rank], W1[L - 1][rank]
        s = torch.zeros(1, dtype=torch.float64)
        if rank > 0:
            dist.recv(s, rank - 1)
        acc = float(s[0])
        for v in t[w0:w1].ravel():
            acc = acc + float(v)
        s[0] = acc
        if rank + 1 < world:
            dist.send(s, rank + 1)
        dist.broadcast(s, world - 1)
        want = o.dot(t.ravel(), np.ones(t.size))
        out[rank] = (float(s[0]) == want, float(s[0]), want)
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 3])
def test_row_slab_host_logic_gloo(world):
    port = free_port()
    mgr = mp.Manager()
    out = mgr.dict()
    mp.spawn(_worker, args=(world, port, out), nprocs=world, join=True)
    assert len(out) == world
    for r in range(world):
        assert out[r][0], out[r]
