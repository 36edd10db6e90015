"""Per-(kernel family, level) milliseconds of one cycle of a workload (best of 3 profiled cycles)."""
import collections, json, os, sys
import numpy as np, torch
sys.path.insert(0, os.getcwd())
import bench
from paper_0805_3041_b200 import gmg
WL = sys.argv[1] if len(sys.argv) > 1 else "C4"
w = bench.WORKLOADS[WL]
p = gmg.MultilevelProblem(*bench.wl_args(w))
n = p.n(w["levels"])
b = torch.from_numpy(gmg.random_vector(n, 1)).cuda()
x = torch.from_numpy(np.zeros(n) if not w["seed_x"] else gmg.random_vector(n, w["seed_x"])).cuda()
spec = gmg.CycleSpec(smoother="jacobi", smoothing_omega=0.7, pre_steps=w["pre"], post_steps=w["post"], tolerance=1e-300, max_cycles=30)
best = None
for rep in range(3):
    prof = gmg.profile_cycle(p, spec, b.data_ptr(), x.data_ptr(), skip=0)
    fam = collections.defaultdict(float)
    for e in prof: fam[(e["kernel"], e["level"])] += e["ms"]
    if best is None: best = dict(fam)
    else:
        for k in fam: best[k] = min(best[k], fam[k])
for k in sorted(best): print(json.dumps([k[0], k[1], round(best[k], 4)]))
