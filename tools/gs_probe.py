"""Gauss-Seidel wavefront probe: smooth_step (defect + k_gs_wave) on the finest level of a
1023^2 (levels=10) or 2047^2 (levels=11) grid, host round trips excluded by the profile API.

    python tools/gs_probe.py [levels] [alpha] [steps]
"""
import os, sys
import numpy as np
import torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_0805_3041_b200 import gmg

L = int(sys.argv[1]) if len(sys.argv) > 1 else 10
alpha = float(sys.argv[2]) if len(sys.argv) > 2 else 1e-2
s = int(sys.argv[3]) if len(sys.argv) > 3 else 1
p = gmg.MultilevelProblem(L, alpha=alpha)
n = p.n(L)
b = torch.from_numpy(gmg.random_vector(n, 1)).cuda()
x = torch.from_numpy(gmg.random_vector(n, 2)).cuda()
spec = gmg.CycleSpec(smoother="gauss_seidel", pre_steps=s, post_steps=s, tolerance=1e-300, max_cycles=3)
for skip in (0, 1):
    prof = gmg.profile_cycle(p, spec, b.data_ptr(), x.data_ptr(), skip=skip)
    tot = sum(e["ms"] for e in prof)
    fam = {}
    for e in prof:
        k = (e["kernel"], e["level"])
        fam[k] = fam.get(k, 0.0) + e["ms"]
    print(f"cycle {skip + 1}: {tot:.3f} ms in {len(prof)} launches")
    for k, v in sorted(fam.items(), key=lambda kv: -kv[1])[:8]:
        print(f"   {k[0]:28s} L{k[1]:2d} {v:8.3f} ms")
