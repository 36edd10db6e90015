"""Repeated ILU(0) smooth_step on a one-row level (debug probe for compute-sanitizer)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "oracle"))
import numpy as np
from paper_0805_3041_b200 import gmg
from pyoracle import Oracle
a = (3, 60, 1, (1.0, 1.02), "cartesian", 0.5, 2.0)
o = Oracle(*a)
x = Oracle.random_vector(60, 61)
b = Oracle.random_vector(60, 71)
want = o.smooth_step(1, "ilu0", 1.0, 1.0, x, b)
d = gmg.MultilevelProblem(*a)
got = gmg.smooth_step(d, 1, "ilu0", 1.0, x, b, 1.0)
print("equal", np.array_equal(got, want))
