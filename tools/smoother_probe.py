"""Times the finest-level smoother kernel variants (gmg_dev_time_smoother) over a
matrix of anisotropy and fused step counts, and launches each once for ncu.

    python tools/smoother_probe.py [--levels 13] [--alphas 1,1e-2] [--steps 1,2,3,4] [--reps 10]
"""
import argparse
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_0805_3041_b200 import gmg  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--levels", type=int, default=13)
ap.add_argument("--alphas", default="1,1e-2")
ap.add_argument("--steps", default="1,2,3,4")
ap.add_argument("--variants", default="0,1,2")
ap.add_argument("--reps", type=int, default=10)
a = ap.parse_args()
names = {0: "from P e", 1: "u + w P uc", 2: "from u"}
for alpha in [float(x) for x in a.alphas.split(",")]:
    p = gmg.MultilevelProblem(a.levels, 1, 1, (1.0, 1.0), "cartesian", alpha, 1.0)
    for m in [int(x) for x in a.steps.split(",")]:
        for v in [int(x) for x in a.variants.split(",")]:
            ms, by = gmg.time_smoother(p, gmg.CycleSpec(smoother="jacobi", pre_steps=m, post_steps=m), variant=v,
                                       reps=a.reps)
            print(f"alpha={alpha:g} M={m} {names[v]:>11}: {ms:.3f} ms, {by / ms / 1e6:.0f} GB/s", flush=True)
    p.close()
