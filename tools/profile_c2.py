import os, sys
import numpy as np
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_0805_3041_b200 import gmg
p = gmg.MultilevelProblem(10, alpha=1e-2)
n = p.n(10)
b = gmg.random_vector(n, 1)
x = gmg.random_vector(n, 2)
s = int(sys.argv[1]) if len(sys.argv) > 1 else 1
r = gmg.solve(p, b, gmg.CycleSpec(smoother="gauss_seidel", pre_steps=s, post_steps=s, tolerance=1e-30, max_cycles=2), x)
print(r.residual_history)
