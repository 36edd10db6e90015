"""Exact-sum engine phase counters per problem size: where a walk CTA's cycles go.

    python tools/walk_phases.py [levels ...]
"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
from paper_0805_3041_b200 import gmg  # noqa: E402

for L in [int(a) for a in sys.argv[1:]] or [8, 9, 10, 11, 13]:
    p = gmg.MultilevelProblem(L)
    n = p.n(L)
    b = gmg.random_vector(n, 1)
    x = np.zeros(n)
    spec = gmg.CycleSpec(smoother="jacobi", tolerance=1e-300, max_cycles=3)
    gmg.seqsum_stats(p, reset=True)
    gmg.solve(p, b, spec, x)
    st = gmg.seqsum_stats(p)
    ctas = max(st["walk_ctas"], 1)
    ph = {k: st[k] / ctas for k in ("walk_load", "walk_prefix_lookback", "walk_thread_walk",
                                      "walk_block_merge", "walk_run_lookback")}
    print(f"L={L} sums={st['sums']} ctas={ctas} records={st['records']} rewalks={st['rewalks']} "
          f"dense_chunks={st['dense_chunks']} chain cyc/rec={st['chain_cycles'] / max(st['records'], 1):.0f}")
    print("   per-CTA cycles: " + ", ".join(f"{k[5:]}={v:.0f}" for k, v in ph.items()))
