"""The drop-in story end to end: the reference's own gmg::solve and
gmg_b200::solve (include/gmg_b200.hpp over the C ABI) on the same reference
objects must agree bit for bit, as must gmg::make_start_vector / run_study and
their device versions (every sweep solve on the GPU), and problems rebuilt in
the same stack slot with other alpha / level counts must never reuse stale
device operators (oracle/shim_demo.cpp, built from the reference
sources into oracle/_ref/ where /root/reference exists; the binary travels)."""
import json
import os
import subprocess

import pytest

from conftest import ROOT

DEMO = os.path.join(ROOT, "oracle", "_ref", "shim_demo")


@pytest.mark.gpu
@pytest.mark.skipif(not os.path.exists(DEMO), reason="oracle/_ref/shim_demo not built (needs the reference sources)")
def test_reference_solve_vs_b200_shim(gpu):
    r = subprocess.run([DEMO], capture_output=True, text=True, timeout=600)
    lines = [json.loads(l) for l in r.stdout.splitlines() if l.startswith("{")]
    assert len(lines) == 15, r.stdout + r.stderr
    for case in lines:
        assert case["identical"], case
    assert r.returncode == 0, r.stdout + r.stderr
