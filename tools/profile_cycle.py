"""Runs one solve of a workload for profiling (ncu launch lists / full captures).

    python tools/profile_cycle.py [--workload C4] [--cycles 2] [--reduction exact]
"""
import argparse
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402
from paper_0805_3041_b200 import gmg  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--workload", default="C4")
ap.add_argument("--cycles", type=int, default=2)
ap.add_argument("--reduction", default="exact")
a = ap.parse_args()
w = bench.WORKLOADS[a.workload]
p = gmg.MultilevelProblem(w["levels"], 1, 1, (1.0, 1.0), "cartesian", w["alpha"], w["beta"])
n = p.n(w["levels"])
b = gmg.random_vector(n, 1)
x = np.zeros(n) if not w["seed_x"] else gmg.random_vector(n, w["seed_x"])
spec = gmg.CycleSpec(smoother="jacobi", smoothing_omega=0.7, pre_steps=w["pre"], post_steps=w["post"],
                     tolerance=1e-300, max_cycles=a.cycles, reduction=a.reduction)
r = gmg.solve(p, b, spec, x)
print("history", r.residual_history)
