"""Times the C2 configs (1023^2, Gauss-Seidel s+s, eps sweep) on the GPU."""
import os, sys, time
import numpy as np
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_0805_3041_b200 import gmg
for eps in (1.0, 1e-2):
    p = gmg.MultilevelProblem(10, alpha=eps)
    n = p.n(10)
    b = gmg.random_vector(n, 1)
    for s in (1, 2, 4):
        spec = gmg.CycleSpec(smoother="gauss_seidel", pre_steps=s, post_steps=s, tolerance=1e-8, max_cycles=50)
        x = gmg.random_vector(n, 2)
        gmg.solve(p, b, spec, x)
        x = gmg.random_vector(n, 2)
        t0 = time.perf_counter()
        r = gmg.solve(p, b, spec, x)
        dt = time.perf_counter() - t0
        print(f"C2 eps={eps:g} s={s}: {r.iterations} cycles, {1e3*dt/r.iterations:.2f} ms/cycle, "
              f"{n*r.iterations/dt/1e9:.3f} G DOF*cyc/s")
