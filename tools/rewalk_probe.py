import os, sys
import numpy as np
sys.path.insert(0, os.getcwd()); sys.path.insert(0, os.path.join(os.getcwd(), "oracle"))
from paper_0805_3041_b200 import gmg
from pyoracle import Oracle
d = gmg.MultilevelProblem(11)
o = Oracle(6)
def run(name, a):
    gmg.seqsum_stats(d, reset=True)
    got = gmg.norm_l2(d, a); want = o.norm_l2(a)
    g2 = gmg.dot(d, a, np.ones_like(a)); w2 = o.dot(a, np.ones_like(a))
    st = gmg.seqsum_stats(d)
    print(name, got == want, g2 == w2, {k: st[k] for k in ("records", "rewalks", "rewalk_terms", "dense_chunks", "break_adds")})
n = 1 << 20
rng = np.random.default_rng(5)
run("uniform", rng.uniform(-1, 1, n))
run("wide", rng.uniform(-1, 1, n) * 10.0 ** rng.integers(-12, 12, n))
a = rng.uniform(-1, 1, n); a[::4096] = 1e17; a[1::4096] = -1e17
run("cancel", a)
a = np.ones(n) * 2.0**-30; a[n // 3] = 2.0**40; a[2 * n // 3] = -2.0**40
run("spike", a)
a = rng.uniform(-1, 1, n); a = a - a.mean() ; a[:n//2] *= 1e-8
run("tiny-then-big", a)
k = np.arange(n); a = np.where(k % 2 == 0, 1.0, -1.0) * (1 + 2.0**-30 * rng.integers(0, 8, n))
run("alternating", a)
