"""Launch each smoother variant once (for ncu): python tools/smoother_probe.py [levels] [reps]"""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_0805_3041_b200 import gmg

L = int(sys.argv[1]) if len(sys.argv) > 1 else 13
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 1
p = gmg.MultilevelProblem(L)
for variant in (0, 1, 2):
    ms, by = gmg.time_smoother(p, gmg.CycleSpec(smoother="jacobi"), variant=variant, reps=reps)
    print(f"smoother variant {variant}: {ms:.3f} ms, {by/ms/1e6:.0f} GB/s")
