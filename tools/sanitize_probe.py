"""Small device runs for compute-sanitizer (racecheck / synccheck / memcheck):
a Gauss-Seidel wavefront solve (k_gs_wave), an ILU(0) forward/backward wave,
exact-order sums long enough for the walk + scan/chain engine (k_ss_walk,
k_ss_scan_chain), and a Jacobi F-cycle through the warp-strip kernels.

    compute-sanitizer --tool racecheck python tools/sanitize_probe.py
"""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_0805_3041_b200 import gmg  # noqa: E402

p = gmg.MultilevelProblem(8, 1, 1, (1.0, 1.0), "cartesian", 0.1, 1.0)  # 255^2 finest
n = p.n(8)
b = gmg.random_vector(n, 1)
for kind in ("gauss_seidel", "ilu0", "jacobi"):
    x = np.zeros(n)
    r = gmg.solve(p, b, gmg.CycleSpec(smoother=kind, smoother_omega=1.0, tolerance=1e-30, max_cycles=2), x)
    print(kind, r.iterations, r.residual_history[-1])
v = gmg.random_vector(1 << 18, 3)  # 262144 terms: 256 walk chunks + scan/chain
print("norm", gmg.norm_l2(p, v), "dot", gmg.dot(p, v, v[::-1].copy()))
