"""Per-cycle launch profile across a solve (gmg_dev_profile_cycle): for cycle
k = skip+1 of the workload's solve, the total ms per kernel family, to see how
the data-dependent exact-sum cost moves as the solve converges.

    python tools/cycle_profile.py [--workload C4] [--skips 0,4,8,11,15,19]
"""
import argparse
import collections
import json
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402
from paper_0805_3041_b200 import gmg  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--workload", default="C4")
ap.add_argument("--skips", default="0,4,8,11,15,19")
ap.add_argument("--reduction", default="exact")
a = ap.parse_args()
w = bench.WORKLOADS[a.workload]
p = gmg.MultilevelProblem(*bench.wl_args(w))
n = p.n(w["levels"])
b = torch.from_numpy(gmg.random_vector(n, 1)).cuda()
x0 = np.zeros(n) if not w["seed_x"] else gmg.random_vector(n, w["seed_x"])
x = torch.from_numpy(x0).cuda()
spec = gmg.CycleSpec(smoother="jacobi", smoothing_omega=0.7, pre_steps=w["pre"], post_steps=w["post"],
                     tolerance=1e-300, max_cycles=30, reduction=a.reduction)
out = {}
for skip in [int(s) for s in a.skips.split(",")]:
    prof = gmg.profile_cycle(p, spec, b.data_ptr(), x.data_ptr(), skip=skip)
    fam = collections.defaultdict(float)
    for e in prof:
        fam[e["kernel"]] += e["ms"]
    out[skip + 1] = dict(total_ms=round(sum(fam.values()), 3), **{k: round(v, 3) for k, v in sorted(fam.items())})
    print(json.dumps({"cycle": skip + 1, **out[skip + 1]}), flush=True)
