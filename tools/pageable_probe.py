"""Pageable-buffer solve through gmg_dev_solve (what the C++ shim does with std::vector storage):
C4, 12 cycles to the reference tolerance, with the staged pinned-ring transfer (default) or the
runtime's pageable copy (GMG_NO_STAGE=1). Prints DOF*cycles/s end to end and sha256 of x."""
import hashlib
import os
import sys
import time

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402
from paper_0805_3041_b200 import gmg  # noqa: E402

w = bench.WORKLOADS["C4"]
prob = gmg.MultilevelProblem(*bench.wl_args(w, 1), device=0)
n = prob.n(w["levels"])
b = gmg.random_vector(n, 1)
spec = gmg.CycleSpec(tolerance=w["tol"], max_cycles=50, smoother="jacobi", smoother_omega=1.0,
                     smoothing_omega=0.7, pre_steps=w["pre"], post_steps=w["post"], cycle="F",
                     adaptive_correction=True, reduction="exact")
for rep in range(3):
    x = np.zeros(n)
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    r = gmg.solve(prob, b, spec, x)
    dt = time.perf_counter() - t0
    print(f"stage={'off' if os.environ.get('GMG_NO_STAGE') else 'on'} rep {rep}: {r.iterations} cycles, "
          f"{dt * 1e3:.1f} ms, {n * r.iterations / dt / 1e9:.3f} G DOF*cycles/s, "
          f"x sha256 {hashlib.sha256(x.tobytes()).hexdigest()[:16]}")
