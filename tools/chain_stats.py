"""Exact-sum engine counters for one late C4 cycle: solve 9 cycles, reset, run 1 more."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
from paper_0805_3041_b200 import gmg

L = int(sys.argv[1]) if len(sys.argv) > 1 else 13
warm = int(sys.argv[2]) if len(sys.argv) > 2 else 9
p = gmg.MultilevelProblem(L)
n = p.n(L)
b = torch.from_numpy(gmg.random_vector(n, 1)).cuda()
x = torch.zeros(n, dtype=torch.float64, device="cuda")
spec = gmg.CycleSpec(smoother="jacobi", tolerance=1e-300, max_cycles=warm)
gmg.solve_device(p, b.data_ptr(), x.data_ptr(), spec)
gmg.seqsum_stats(p, reset=True)
spec1 = gmg.CycleSpec(smoother="jacobi", tolerance=1e-300, max_cycles=1)
r = gmg.solve_device(p, b.data_ptr(), x.data_ptr(), spec1)
st = gmg.seqsum_stats(p)
print("wall ms", 1e3 * r.wall_seconds)
for k, v in st.items():
    print(f"  {k:22s} {v}")
if st["records"]:
    print("chain cycles/record %.0f, excl rewalk %.0f" % (st["chain_cycles"] / st["records"],
          (st["chain_cycles"] - st["rewalk_cycles"]) / st["records"]))
