"""Uninitialised-memory probe: dirty the device heap with NaNs, then run the
smoother parity on fresh problems and report mismatching kinds."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "oracle"))
import numpy as np
import torch
from paper_0805_3041_b200 import gmg
from pyoracle import Oracle

t = torch.full((int(sys.argv[1]) if len(sys.argv) > 1 else 2_000_000_000,), float("nan"), dtype=torch.float64,
               device="cuda")
torch.cuda.synchronize()
del t
torch.cuda.empty_cache()
GE = [(3, 60, 1, (1.0, 1.02), "cartesian", 0.5, 2.0), (5, 1, 1, (1.0, 1.0), "cartesian", 1.0, 1.0),
      (4, 3, 2, (1.1, 0.93), "spherical", 1.3, 0.7)]
bad = 0
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 1
for a in GE * reps:
    d, o = gmg.MultilevelProblem(*a), Oracle(*a)
    for l in range(1, d.num_levels + 1):
        n = d.n(l)
        x = Oracle.random_vector(n, 60 + l)
        b = Oracle.random_vector(n, 70 + l)
        for kind in gmg.SMOOTHERS:
            for som in (1.0, 0.6):
                for damp in (0.7, 1.0):
                    got = gmg.smooth_step(d, l, kind, som, x, b, damp)
                    want = o.smooth_step(l, kind, som, damp, x, b)
                    if not np.array_equal(got.view(np.uint64), want.view(np.uint64)):
                        nz = np.nonzero(got != want)[0]
                        print("MISMATCH", a[:3], l, kind, som, damp, len(nz), nz[:5], got[nz[:2]], want[nz[:2]])
                        bad += 1
print("bad", bad)
