"""Out-of-bounds regression: the device path under GMG_GUARD_ALLOC (every device
buffer in its own virtual-address reservation, flush against unmapped guard
pages, csrc/dalloc.h), so any read or write past a buffer faults instead of
landing in a neighbouring allocation. Covers the operator classes whose
coefficient tables are read per point (ROWX, FIELD), the streaming kernels'
halo columns and rows, row slabs and the exact-sum engine (both chunk sizes).
"""
import os
import subprocess
import sys

import pytest

from conftest import ROOT

pytestmark = pytest.mark.gpu

SCRIPT = r'''
import sys, numpy as np
sys.path.insert(0, ROOT)
from paper_0805_3041_b200 import gmg
cases = [
    ((4, 2, 1, (1.0, 1.0), "cartesian", 0.3, 1.0), None),          # non-dyadic x: ROWX/FIELD
    ((5, 1, 1, (1.05, 0.97), "spherical", 1.0, 0.5), None),         # FIELD
    ((6, 1, 1, (1.0, 1.0), "cylindrical", 1.0, 1.0), None),         # ROWX
    ((7, 2, 1, (1.0, 1.0), "cartesian", 0.3, 1.0), 3),               # row slabs, small-chunk sums
    ((9, 1, 1, (1.0, 1.0), "cartesian", 1.0, 1.0), None),           # large-level kernels, walk/chain
]
for args, world in cases:
    L = args[0]
    p = gmg.MultilevelProblem(*args, slabs=gmg.Slabs(world=world, min_rows=15) if world else None)
    n = p.n(L)
    b = gmg.random_vector(n, 1)
    x = gmg.random_vector(n, 2)
    if not world:
        for l in range(1, L + 1):
            v = gmg.random_vector(p.n(l), 3)
            gmg.apply(p, l, v)
            gmg.residual(p, l, v, v)
            gmg.smooth_step(p, l, "jacobi", 1.0, v, v, 0.7)
            if l >= 2:
                gmg.restriction(p, l, v)
    for pre, post in [(2, 2), (3, 5)]:
        spec = gmg.CycleSpec(smoother="jacobi", pre_steps=pre, post_steps=post, tolerance=1e-30, max_cycles=3)
        gmg.solve(p, b, spec, x.copy())
print("guard ok")
'''


def test_device_path_has_no_out_of_bounds_access(gpu):
    env = dict(os.environ, GMG_GUARD_ALLOC="1")
    for mode in ("1", "2"):  # buffer flush against the end, then the start, of its mapping
        env["GMG_GUARD_ALLOC"] = mode
        r = subprocess.run([sys.executable, "-c", f"ROOT = {ROOT!r}\n" + SCRIPT], env=env, capture_output=True,
                           text=True, timeout=600)
        assert r.returncode == 0 and "guard ok" in r.stdout, (mode, r.stdout[-2000:], r.stderr[-2000:])
