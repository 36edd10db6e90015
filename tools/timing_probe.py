"""Where does a cycle's wall time go? Compares solve timings across reduction modes and sizes."""
import os, sys, time
import numpy as np
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_0805_3041_b200 import gmg

L = int(sys.argv[1]) if len(sys.argv) > 1 else 13
p = gmg.MultilevelProblem(L)
n = p.n(L)
b = torch.from_numpy(gmg.random_vector(n, 1)).cuda()
x = torch.zeros(n, dtype=torch.float64, device="cuda")
for red in ["exact", "fast"]:
    for cyc in [1, 5]:
        spec = gmg.CycleSpec(smoother="jacobi", tolerance=1e-300, max_cycles=cyc, reduction=red)
        gmg.solve_device(p, b.data_ptr(), x.data_ptr(), spec)
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        r = gmg.solve_device(p, b.data_ptr(), x.data_ptr(), spec)
        torch.cuda.synchronize()
        dt = time.perf_counter() - t0
        print(f"L={L} {red:5s} cycles={cyc}: {1e3*dt:8.2f} ms total, wall in report {1e3*r.wall_seconds:8.2f}")
        if red == "exact":
            print("   engine stats (warm+timed calls):", gmg.seqsum_stats(p))
for variant in (0, 1, 2):
    ms, by = gmg.time_smoother(p, gmg.CycleSpec(smoother="jacobi"), variant=variant, reps=10)
    print(f"smoother variant {variant}: {ms:.3f} ms, {by/ms/1e6:.0f} GB/s")
