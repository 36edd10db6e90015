"""One Gauss-Seidel smooth_step on the finest level (for an ncu capture of k_gs_wave): python tools/gs_step.py [levels] [alpha]"""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_0805_3041_b200 import gmg
L = int(sys.argv[1]) if len(sys.argv) > 1 else 10
alpha = float(sys.argv[2]) if len(sys.argv) > 2 else 1e-2
p = gmg.MultilevelProblem(L, alpha=alpha)
n = p.n(L)
y = gmg.smooth_step(p, L, "gauss_seidel", 1.0, gmg.random_vector(n, 2), gmg.random_vector(n, 1), 1.0)
print(float(y[0]), float(y[-1]))
