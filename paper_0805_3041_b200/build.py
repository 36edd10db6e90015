"""In-tree build of libgmg_b200.so (sm_100a) — no JIT caches, so the built
library travels to the GPU box with the repo snapshot.

    python -m paper_0805_3041_b200.build [--force]
"""
from __future__ import annotations

import os
import subprocess
import sys

PKG = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(PKG)
CSRC = os.path.join(PKG, "csrc")
# GMG_LIB_OUT / GMG_BUILD_DIR: an alternative build (e.g. an instrumented -D variant for A/B
# timing) next to the product library; load it with GMG_LIB_PATH.
BUILD = os.environ.get("GMG_BUILD_DIR") or os.path.join(ROOT, "build", "gmg_b200")
LIB = os.environ.get("GMG_LIB_OUT") or os.path.join(PKG, "libgmg_b200.so")

NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
# -fmad=false: no FMA contraction anywhere (bit-exact with the reference's
# unfused x86-64 arithmetic); -ffp-contract=off for the host code likewise.
# No -split-compile: it cost 6% per C4 cycle (worse code for the streaming kernels) and made
# builds of the same source differ by +-3% (kernel placement depends on its worker threads);
# the library builds as parallel translation units instead (inst.h).
# -static-global-template-stub=false: kernels instantiated in one translation unit (inst.cu) are
# launched from another (solver.cu, extern template) through their host stubs.
NVFLAGS = ["-O3", "-std=c++17", *ARCH, "-lineinfo", "-fmad=false", "--expt-relaxed-constexpr",
           "-static-global-template-stub=false", "-diag-suppress", "20279,20281",
           "-Xcompiler", "-fPIC,-ffp-contract=off,-fno-fast-math", "-Xptxas", "-v"]
CXXFLAGS = ["-O2", "-std=c++17", "-fPIC", "-ffp-contract=off", "-fno-fast-math", "-Wall"]

SOURCES_CU = ["solver.cu"]
INST_GROUPS = [1, 2, 3, 4]  # inst.cu, once per group of inst.h
SOURCES_CPP = ["host_setup.cpp"]
def _deps():
    """Every header the sources may include (all of csrc/ plus the C ABI)."""
    hs = [os.path.join(CSRC, f) for f in os.listdir(CSRC) if f.endswith((".cuh", ".h", ".hpp"))]
    return hs + [os.path.join(ROOT, "include", "gmg_b200.h"), os.path.abspath(__file__)]  # (flags live here)


def _newer(target: str, sources) -> bool:
    if not os.path.exists(target):
        return True
    t = os.path.getmtime(target)
    return any(os.path.getmtime(s) > t for s in sources)


def _run(cmd, log):
    r = subprocess.run(cmd, capture_output=True, text=True)
    with open(log, "w") as f:
        f.write(" ".join(cmd) + "\n" + r.stdout + r.stderr + "\n")
    if r.returncode != 0:
        sys.stderr.write(r.stdout + r.stderr)
        raise RuntimeError(f"build failed: {' '.join(cmd[:3])} ... (see {log})")


def build(force: bool = False, verbose: bool = False) -> str:
    os.makedirs(BUILD, exist_ok=True)
    log = os.path.join(BUILD, "build.log")
    deps = _deps()
    objs = []
    extra = os.environ.get("GMG_EXTRA_NVFLAGS", "").split()  # e.g. -DGMG_KDEBUG (debug builds)
    jobs = []  # (name, command, object): the CUDA translation units compile in parallel
    for src in SOURCES_CU:
        s = os.path.join(CSRC, src)
        o = os.path.join(BUILD, src + ".o")
        if force or _newer(o, [s, *deps]):
            jobs.append((src, [NVCC, *NVFLAGS, *extra, "-c", s, "-o", o], o))
        objs.append(o)
    for g in INST_GROUPS:
        s = os.path.join(CSRC, "inst.cu")
        o = os.path.join(BUILD, f"inst{g}.o")
        if force or _newer(o, [s, *deps]):
            jobs.append((f"inst.cu[{g}]", [NVCC, *NVFLAGS, *extra, f"-DGMG_INST_GROUP={g}", "-c", s, "-o", o], o))
        objs.append(o)
    if jobs:
        from concurrent.futures import ThreadPoolExecutor
        if verbose:
            print("nvcc", ", ".join(j[0] for j in jobs), flush=True)
        with ThreadPoolExecutor(max_workers=len(jobs)) as ex:
            list(ex.map(lambda j: _run(j[1], j[2] + ".log"), jobs))
    for src in SOURCES_CPP:
        s = os.path.join(CSRC, src)
        o = os.path.join(BUILD, src + ".o")
        if force or _newer(o, [s, *deps]):
            if verbose:
                print("g++", src, flush=True)
            _run(["g++", *CXXFLAGS, "-c", s, "-o", o], o + ".log")
        objs.append(o)
    if force or _newer(LIB, objs):
        _run([NVCC, "-shared", *ARCH, "-Xcompiler", "-fPIC", *objs, "-o", LIB], log)
    return LIB


if __name__ == "__main__":
    print(build(force="--force" in sys.argv, verbose=True))
