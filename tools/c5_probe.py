"""C5 (16383^2, eps=1e-2, jacobi 3+3, random start) timing + exact-sum engine counters."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_0805_3041_b200 import gmg
L = int(sys.argv[1]) if len(sys.argv) > 1 else 14
p = gmg.MultilevelProblem(L, alpha=1e-2)
n = p.n(L)
b = torch.from_numpy(gmg.random_vector(n, 1)).cuda()
x = torch.from_numpy(gmg.random_vector(n, 2)).cuda()
for red in ["exact", "fast"]:
    spec = gmg.CycleSpec(smoother="jacobi", pre_steps=3, post_steps=3, tolerance=1e-300, max_cycles=2, reduction=red)
    gmg.seqsum_stats(p)
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    r = gmg.solve_device(p, b.data_ptr(), x.data_ptr(), spec)
    torch.cuda.synchronize()
    print(f"L={L} {red}: {1e3*(time.perf_counter()-t0)/2:.1f} ms/cycle", r.residual_history)
    print("   ", gmg.seqsum_stats(p))
