"""Deviation of the tree-order ("fast") reduction mode from the reference's golden histories:
max over cycles of |r_k(fast) - r_k(ref)| / r_k(ref), and the iteration counts."""
import os
import sys
import time

import numpy as np

sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tests"))
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from test_gpu_parity import run_fixture, unhex  # noqa: E402
from paper_0805_3041_b200 import gmg  # noqa: E402

for name in sys.argv[1:] or ["c1_adaptive", "c4_small_2047", "c3p_cylindrical", "c4_adaptive", "c5_10cycle"]:
    g, d, b, x, spec = run_fixture(name, {"reduction": "fast"})
    t0 = time.perf_counter()
    rep = gmg.solve(d, b, spec, x)
    dt = time.perf_counter() - t0
    want = np.array(unhex(g["history"]))
    got = np.array(rep.residual_history)
    m = min(len(want), len(got))
    dev = np.abs(got[:m] - want[:m]) / want[:m]
    print(f"{name}: iterations {rep.iterations} (ref {g['iterations']}), max rel dev {dev.max():.3e} "
          f"at cycle {int(dev.argmax())}, per cycle {['%.1e' % v for v in dev]}, {dt:.2f} s")
    del d
