"""Multi-process row slabs over NCCL: one process
per GPU, halos / threshold gathers / the rank-ordered exact-sum handoff over
NCCL. Needs >= 2 GPUs (NCCL refuses two ranks on one device); on one GPU the
same schedule is covered by the virtual-rank tests (test_gpu_slabs.py) and the
host logic by the gloo tests (test_dist_host.py)."""
import json
import os
import subprocess
import sys

import pytest

from conftest import ROOT

pytestmark = pytest.mark.gpu


def n_gpus():
    try:
        import torch
        return torch.cuda.device_count()
    except Exception:
        return 0


@pytest.mark.skipif(n_gpus() < 2, reason="needs >= 2 GPUs")
@pytest.mark.parametrize("world", [2, 4, 8])
def test_nccl_row_slabs_bitexact(world):
    if n_gpus() < world:
        pytest.skip(f"needs {world} GPUs")
    import socket
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        port = s.getsockname()[1]
    env = dict(os.environ, NCCL_DEBUG="INFO", NCCL_DEBUG_SUBSYS="INIT", NCCL_DEBUG_FILE="/dev/stderr")
    r = subprocess.run([sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={world}",
                        "--master-addr", "127.0.0.1", f"--master-port={port}",
                        os.path.join(ROOT, "tests", "helpers", "nccl_slab_worker.py")],
                       capture_output=True, text=True, timeout=900, env=env)
    lines = [json.loads(l) for l in r.stdout.splitlines() if l.startswith("{")]
    assert len(lines) == 3, r.stdout[-3000:] + r.stderr[-3000:]
    for c in lines:
        assert c["identical"] and c["world"] == world, c
    assert r.returncode == 0, r.stderr[-3000:]


@pytest.mark.skipif(n_gpus() < 2, reason="needs >= 2 GPUs")
def test_bench_gpus_2_spawns_ranks():
    r = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--gpus", "2", "--steps", "3", "--warmup", "3",
                        "--workload", "C4", "--no-cpu-baseline", "--no-c5", "--e2e-steps", "1"],
                       capture_output=True, text=True, timeout=900)
    lines = [json.loads(l) for l in r.stdout.splitlines() if l.startswith("{")]
    assert r.returncode == 0 and len(lines) == 1, r.stdout[-2000:] + r.stderr[-2000:]
    assert lines[0]["n_gpus"] == 2 and lines[0]["scaling"] == "strong"
