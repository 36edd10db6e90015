"""One rank of the multi-process row-slab solve (NCCL transport, one GPU per
rank), launched by tests/test_gpu_multi.py under torch.distributed.run.

Every rank builds its slab of the same problem over a shared NCCL group and
solves; rank 0 also solves the single-domain problem and compares the residual
history and the gathered solution bit for bit. Exit status 0 = identical."""
import json
import os
import sys

import numpy as np
import torch
import torch.distributed as dist

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)
from paper_0805_3041_b200 import gmg  # noqa: E402

CASES = [
    # name, problem args, spec, seed_x
    ("C4-small 2047^2 F jacobi 2+2 adaptive", (11, 1, 1, (1.0, 1.0), "cartesian", 1.0, 1.0),
     dict(smoother="jacobi", smoothing_omega=0.7, tolerance=1e-10, max_cycles=6), 0),
    ("1023^2 eps=1e-2 3+3 random start (walk/chain engine per slab)", (10, 1, 1, (1.0, 1.0), "cartesian", 1e-2, 1.0),
     dict(smoother="jacobi", smoothing_omega=0.7, pre_steps=3, post_steps=3, tolerance=1e-30, max_cycles=4), 2),
    ("511^2 cylindrical W-cycle 5+6 (multi-launch smoothing)", (9, 1, 1, (1.0, 1.0), "cylindrical", 1.0, 1.0),
     dict(cycle="W", smoother="jacobi", pre_steps=5, post_steps=6, tolerance=1e-9, max_cycles=5), 0),
]


def main():
    rank, world, local = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"]), int(os.environ["LOCAL_RANK"])
    torch.cuda.set_device(local)
    dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    bad = 0
    for name, args, spec_kw, seed_x in CASES:
        ids = [gmg.unique_id() if rank == 0 else None]
        dist.broadcast_object_list(ids, src=0)
        slab = gmg.MultilevelProblem(*args, device=local,
                                     slabs=gmg.Slabs(world=world, rank=rank, min_rows=255, nccl_id=ids[0]))
        r, w, Ls = slab.dist_info()
        L = slab.num_levels
        n = slab.n(L)
        b = gmg.random_vector(n, 1)
        x0 = gmg.random_vector(n, seed_x) if seed_x else np.zeros(n)
        spec = gmg.CycleSpec(**spec_kw)
        xd = x0.copy()
        rd = gmg.solve(slab, b, spec, xd)
        if rank == 0:
            single = gmg.MultilevelProblem(*args, device=local)
            xs = x0.copy()
            rs = gmg.solve(single, b, spec, xs)
            ok = (rs.iterations == rd.iterations and
                  np.array_equal(np.array(rs.residual_history), np.array(rd.residual_history)) and
                  np.array_equal(xs, xd))
            bad += 0 if ok else 1
            print(json.dumps({"case": name, "world": w, "first_sharded_level": Ls, "levels": L,
                              "identical": bool(ok), "cycles": rd.iterations}), flush=True)
            single.close()
        slab.close()
        dist.barrier()
    t = torch.tensor([bad], device="cuda")
    dist.all_reduce(t)
    dist.destroy_process_group()
    sys.exit(1 if int(t.item()) else 0)


if __name__ == "__main__":
    main()
