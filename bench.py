"""Benchmark: fine-grid DOF * F-cycles / s of the B200 multigrid F-cycle.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]
                    [--workload C4|C5|C1|C3p] [--no-cpu-baseline]

A step is one F-cycle (BASELINE.json metric) on workload C4 by default:
8191^2 interior unknowns (8193^2 vertices), 13 levels, -Laplace u = f,
f ~ U[-1,1] from std::mt19937(1), zero start, damped Jacobi 0.7 with 2+2 steps,
adaptive correction weights, exact-order (reference-identical) reductions.
Every vector is 537 MB, far larger than the 126 MB L2, so no L2 flush is needed.

value  : device-resident — b and x already in HBM; K cycles of one solve call,
         timed with CUDA events on the solver stream (max over ranks).
e2e    : through the public C-ABI solve (gmg_dev_solve) with pinned host buffers:
         every step uploads b and x, solves to the reference's tolerance and
         downloads x; wall time of the call; DOF*cycles/s.
roofline: the finest-level post-smoother (u + omega*P uc, 2 Jacobi steps fused)
         timed live with CUDA events; 26 B per fine DOF of algorithmic traffic.
cpu_baseline: the reference compiled from its own sources (oracle/_ref), one
         F-cycle of the same workload on one host core (the reference has no
         intra-solve parallelism).
--impl reference: the same metric from the reference's CPU code on all usable
         host cores (independent solves in parallel threads), rank 0 only.
Multi-GPU (N>1 via torchrun): by default the one grid is split into row slabs
(--parallel slabs): levels with >= 255 interior rows are sharded
over the ranks, halos and the rank-ordered exact reductions go over NCCL, the
coarse levels are replicated. Strong scaling; value = the grid's DOF*cycles/s.
--parallel replicas runs one independent copy of the workload per rank (weak).
Timing = max over ranks either way. `--gpus N` without torchrun re-launches this
script under torch.distributed.run with N ranks (127.0.0.1); under torchrun it
must agree with WORLD_SIZE. NCCL logs its communicator setup (NCCL_DEBUG=INFO,
subsystem INIT) to stderr.
per_level: one extra cycle with CUDA events around every launch
         (gmg_dev_profile_cycle): GB/s and HBM fraction per kernel family and
         level from §8d's algorithmic bytes; levels whose per-launch traffic fits
         in L2 are flagged l2_resident (their GB/s is not an HBM number).
c5     : BASELINE config 5 (16383^2, 14 levels, eps=1e-2, 3+3, random f and x0,
         exactly 10 F-cycles) device-resident on the same GPU, with its own
         per-level table (--no-c5 skips it).
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

WORKLOADS = {
    # name: levels, coarse, alpha, beta, smoothing steps, tol, seed_x
    "C4": dict(levels=13, alpha=1.0, beta=1.0, pre=2, post=2, tol=1e-10, seed_x=0,
               desc="8191^2 interior (8193^2 vertices), 13 levels, isotropic Poisson, jacobi 0.7 2+2, "
                    "F-cycle, adaptive omega_l, exact-order reductions"),
    "C5": dict(levels=14, alpha=1e-2, beta=1.0, pre=3, post=3, tol=1e-30, seed_x=2,
               desc="16383^2 interior (16385^2 vertices), 14 levels, anisotropic eps=1e-2, jacobi 0.7 3+3, "
                    "F-cycle, adaptive omega_l, exact-order reductions"),
    "C1": dict(levels=7, alpha=1.0, beta=1.0, pre=2, post=2, tol=1e-8, seed_x=0,
               desc="127^2 interior (129^2 vertices), 7 levels, isotropic Poisson, jacobi 0.7 2+2"),
    # BASELINE config 3 (no reference counterpart: the oracle restatement is the checker)
    "C3": dict(levels=10, alpha=1.0, beta=1.0, pre=2, post=2, tol=1e-8, seed_x=0, coords="polar", cny=2,
               desc="polar Poisson 1023 (r in [0.1,1], Dirichlet) x 1024 (theta, periodic), 10 levels, "
                    "jacobi 0.7 2+2, F-cycle, adaptive omega_l, exact-order reductions"),
    # SURVEY.md §8(e) weak-scaling family: coarse 15 x (2P-1), 11 levels -> 16383 x (2048P-1) interior
    # (P = 8: exactly the C5 grid, with a 225-unknown level-1 factor); C5's physics and smoother
    "W": dict(levels=11, alpha=1e-2, beta=1.0, pre=3, post=3, tol=1e-30, seed_x=2, cnx=15, cny_per_rank=True,
              desc="weak-scaling family 16383 x (2048P-1) interior, coarse 15 x (2P-1), 11 levels, eps=1e-2, "
                   "jacobi 0.7 3+3, F-cycle, adaptive omega_l, exact-order reductions"),
}


def wl_args(w, world=1):
    """MultilevelProblem / Oracle constructor arguments of a workload (world: ranks, for W)."""
    cny = 2 * world - 1 if w.get("cny_per_rank") else w.get("cny", 1)
    return (w["levels"], w.get("cnx", 1), cny, (1.0, 1.0), w.get("coords", "cartesian"), w["alpha"], w["beta"])


def common_config(wl, n):
    """The config both arms report (identical keys and values)."""
    w = WORKLOADS[wl]
    return {"workload": f"{wl}: {w['desc']}", "dof": n, "reduction": "exact",
            "l2": "inputs larger than L2 (537 MB per vector at C4, 2.1 GB at C5, vs 126 MB L2); no flush"}


def host_info():
    model = "unknown"
    try:
        with open("/proc/cpuinfo") as f:
            for line in f:
                if line.startswith("model name"):
                    model = line.split(":", 1)[1].strip()
                    break
    except OSError:
        pass
    return {"cpu_model": model, "nproc": os.cpu_count(), "affinity_cpus": len(os.sched_getaffinity(0))}


def free_port():
    import socket
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def maybe_spawn(args):
    """--gpus N (N > 1) outside torchrun: re-run this script as N ranks under
    torch.distributed.run on 127.0.0.1 and exit with its status."""
    ws_env = os.environ.get("WORLD_SIZE")
    if ws_env is not None:
        if args.gpus is not None and int(ws_env) != args.gpus:
            sys.exit(f"bench.py: --gpus {args.gpus} disagrees with WORLD_SIZE={ws_env}")
        return
    if args.gpus is None or args.gpus <= 1 or args.impl == "reference":
        return
    import torch
    if torch.cuda.device_count() < args.gpus:
        sys.exit(f"bench.py: --gpus {args.gpus} needs {args.gpus} GPUs, this node has {torch.cuda.device_count()}")
    env = dict(os.environ)
    env.setdefault("NCCL_DEBUG", "INFO")
    env.setdefault("NCCL_DEBUG_SUBSYS", "INIT")
    env.setdefault("NCCL_DEBUG_FILE", "/dev/stderr")
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={args.gpus}",
           "--master-addr", "127.0.0.1", f"--master-port={free_port()}", os.path.abspath(__file__), *sys.argv[1:]]
    sys.exit(subprocess.run(cmd, env=env).returncode)


def load_peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            pk = json.load(f)
        return float(pk["hbm_gbs"]), "measured (MEASURED_PEAKS.json)"
    except Exception:
        return 6650.0, "fallback (B200_PROFILING.md)"


class ClockSampler:
    """SM clocks and throttle reasons sampled during the timed region: NVML every 5 ms
    (nvidia_ml_py), else nvidia-smi every 0.2 s."""

    Q = ("clocks.sm,clocks.max.sm,clocks_event_reasons.active,clocks_event_reasons.hw_slowdown,"
         "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
         "clocks_event_reasons.sw_power_cap")
    # NVML clocks-event reason bits
    BITS = {"sw_power_cap": 0x4, "hw_slowdown": 0x8, "sw_thermal_slowdown": 0x20, "hw_thermal_slowdown": 0x40}

    def __init__(self, index):
        self.index = index
        self.samples = []  # (sm_mhz, max_mhz, set of reason names)
        self._stop = threading.Event()
        self._t = threading.Thread(target=self._run, daemon=True)
        self._nvml = None
        try:
            import pynvml
            pynvml.nvmlInit()
            self._nvml = (pynvml, pynvml.nvmlDeviceGetHandleByIndex(index))
        except Exception:
            self._nvml = None

    def _sample_nvml(self):
        nv, h = self._nvml
        sm = nv.nvmlDeviceGetClockInfo(h, nv.NVML_CLOCK_SM)
        mx = nv.nvmlDeviceGetMaxClockInfo(h, nv.NVML_CLOCK_SM)
        try:
            bits = nv.nvmlDeviceGetCurrentClocksEventReasons(h)
        except Exception:
            bits = nv.nvmlDeviceGetCurrentClocksThrottleReasons(h)
        return float(sm), float(mx), {k for k, b in self.BITS.items() if bits & b}

    def _sample_smi(self):
        out = subprocess.run(["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.Q}",
                              "--format=csv,noheader,nounits"], capture_output=True, text=True,
                             timeout=5).stdout.strip()
        f = [x.strip() for x in out.split(",")]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        return (float(f[0]), float(f[1]), {names[q] for q in range(4) if len(f) > 3 + q and f[3 + q].lower() == "active"})

    def _run(self):
        while not self._stop.is_set():
            try:
                self.samples.append(self._sample_nvml() if self._nvml else self._sample_smi())
            except Exception:
                pass
            self._stop.wait(0.005 if self._nvml else 0.2)

    def __enter__(self):
        self._t.start()
        return self

    def __exit__(self, *a):
        self._stop.set()
        self._t.join(timeout=10)

    def summary(self):
        if not self.samples:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unavailable"]}
        sm = [s[0] for s in self.samples]
        mx = [s[1] for s in self.samples]
        reasons = sorted(set().union(*[s[2] for s in self.samples]))
        return {"sm_mhz": statistics.median(sm), "sm_max_mhz": max(mx), "reasons": reasons,
                "samples": len(self.samples), "source": "nvml" if self._nvml else "nvidia-smi"}


def dist_env():
    ws = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return ws, rank, local


def cpu_reference_fcycle(wl, threads=1, cycles=1, seconds_cap=None):
    """Times `cycles` F-cycles of the reference (oracle/_ref, else the C port) on
    `threads` independent solves run concurrently. Returns (DOF*cycles/s, info)."""
    sys.path.insert(0, os.path.join(ROOT, "oracle"))
    import pyoracle
    kind = "reference" if pyoracle.Reference.available() else "port"
    B = pyoracle.Reference if kind == "reference" else pyoracle.Oracle
    w = WORKLOADS[wl]
    if w.get("coords") == "polar":
        B, kind = pyoracle.Oracle, "port"
    t0 = time.time()
    prob = B(*wl_args(w))
    n = prob.n(w["levels"])
    b = B.random_vector(n, 1)
    setup = time.time() - t0
    spec = pyoracle.CycleSpec(smoother="jacobi", smoother_omega=1.0, smoothing_omega=0.7, pre_steps=w["pre"],
                              post_steps=w["post"], tolerance=1e-300, max_cycles=cycles)
    xs = [np.zeros(n) if not w["seed_x"] else B.random_vector(n, w["seed_x"]) for _ in range(threads)]
    res = [None] * threads
    cpus = sorted(os.sched_getaffinity(0))

    def run(q):
        # pin this solve's thread to one core (sched_setaffinity(0) is per thread on Linux)
        os.sched_setaffinity(0, {cpus[q % len(cpus)]})
        try:
            res[q] = prob.solve(spec, b, xs[q])
        finally:
            os.sched_setaffinity(0, cpus)

    ts = time.time()
    th = [threading.Thread(target=run, args=(q,)) for q in range(threads)]
    for t in th:
        t.start()
    for t in th:
        t.join()
    dt = time.time() - ts
    return threads * n * cycles / dt, dict(kind=kind, setup_s=round(setup, 2), seconds=round(dt, 2), n=n,
                                           pinned_cpus=[cpus[q % len(cpus)] for q in range(threads)])


def usable_threads(n_dof):
    cores = len(os.sched_getaffinity(0))
    try:
        import psutil
        avail = psutil.virtual_memory().available
    except Exception:
        avail = 32 << 30
    per_solve = 20 * 8 * n_dof  # peak transient of one reference solve (~140 B/DOF measured at C5)
    shared = 60 * n_dof  # operators + b
    by_mem = max(1, int((avail * 0.8 - shared) // per_solve))
    return max(1, min(cores, by_mem))


def run_reference_arm(args):
    ws, rank, _ = dist_env()
    if rank != 0:
        return
    wl = args.workload
    w = WORKLOADS[wl]
    sys.path.insert(0, os.path.join(ROOT, "oracle"))
    import pyoracle
    kind = "reference" if pyoracle.Reference.available() else "port"
    B = pyoracle.Reference if kind == "reference" else pyoracle.Oracle
    if w.get("coords") == "polar":
        B = pyoracle.Oracle  # no reference counterpart for polar coordinates: the oracle port
        kind = "port"
    prob = B(*wl_args(w, ws if ws > 1 else (args.gpus or 1)))
    n = prob.n(w["levels"])
    b = B.random_vector(n, 1)
    P = usable_threads(n) if args.ref_threads <= 0 else args.ref_threads
    spec = pyoracle.CycleSpec(smoother="jacobi", smoother_omega=1.0, smoothing_omega=0.7, pre_steps=w["pre"],
                              post_steps=w["post"], tolerance=1e-300, max_cycles=1)
    xs = [np.zeros(n) if not w["seed_x"] else B.random_vector(n, w["seed_x"]) for _ in range(P)]

    def step():
        th = [threading.Thread(target=prob.solve, args=(spec, b, xs[q])) for q in range(P)]
        for t in th:
            t.start()
        for t in th:
            t.join()

    # one C4 step is ~20 s of CPU work: the run is bounded (at most 3 timed steps after one
    # warm-up step) so that any --steps/--warmup finishes within a couple of minutes
    steps, warmup = max(1, min(args.steps, 3)), min(args.warmup, 1)
    for _ in range(warmup):
        step()
    times = []
    for _ in range(steps):
        t0 = time.time()
        step()
        times.append(time.time() - t0)
    total = sum(times)
    value = P * n * steps / total
    line = {
        "impl": "reference", "metric": "fine-grid DOF*F-cycles/s (fp64)", "value": value,
        "unit": "DOF*cycles/s", "n_gpus": ws if ws > 1 else (args.gpus or 1), "steps": steps, "warmup": warmup,
        "steps_requested": args.steps, "warmup_requested": args.warmup,
        "ms_per_step": 1e3 * total / steps, "higher_is_better": True, "scaling": "weak",
        "vs_baseline": None, "dtype": "f64", "data": "synthetic (seeded U[-1,1] rhs from std::mt19937, as the reference tests)",
        "config": common_config(wl, n),
        "parallelism": f"{P} independent reference solves in parallel host threads",
        "cpu_baseline": {"value": value, "unit": "DOF*cycles/s", "cores": P, "kind": kind, "host": host_info(),
                         "sample": f"each step = 1 F-cycle (gmg::solve, max_cycles=1, incl. its r0/|b| norms) "
                                   f"of {wl} on each of {P} independent solves in parallel threads"},
        "e2e": {"value": value, "unit": "DOF*cycles/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


def per_level_table(prof, peak, l2_bytes):
    """Aggregate gmg.profile_cycle entries per (kernel family, level)."""
    rows = {}
    for e in prof:
        k = (e["kernel"], e["level"])
        r = rows.setdefault(k, dict(kernel=e["kernel"], level=e["level"], launches=0, ms=0.0, bytes=0.0,
                                    max_launch_bytes=0.0))
        r["launches"] += 1
        r["ms"] += e["ms"]
        r["bytes"] += e["bytes"]
        r["max_launch_bytes"] = max(r["max_launch_bytes"], e["bytes"])
    out = []
    for (kern, lev), r in sorted(rows.items(), key=lambda kv: (-kv[0][1], kv[0][0])):
        gbs = r["bytes"] / (r["ms"] / 1e3) / 1e9 if r["ms"] > 0 and r["bytes"] > 0 else None
        out.append({"kernel": kern, "level": lev, "launches": r["launches"], "ms": round(r["ms"], 4),
                    "GBps": None if gbs is None else round(gbs, 1),
                    "frac": None if gbs is None else round(gbs / peak, 3),
                    "l2_resident": bool(0 < r["max_launch_bytes"] <= l2_bytes)})
    total = sum(e["ms"] for e in prof)
    return {"entries": out, "profiled_ms_per_cycle": round(total, 4),
            "how": "cycle 5 of the solve run outside the graph, CUDA events around every launch on the solver "
                   "stream; bytes = "
                   "SURVEY.md 8(d) algorithmic bytes per DOF x level DOFs; ss_* chains carry no streamed bytes"}


def run_c5(gmg, torch, peak, l2_bytes, reduction):
    """BASELINE config 5 exactly: 10 F-cycles device-resident, plus its per-level table."""
    w = WORKLOADS["C5"]
    t0 = time.time()
    prob = gmg.MultilevelProblem(w["levels"], 1, 1, (1.0, 1.0), "cartesian", w["alpha"], w["beta"])
    n = prob.n(w["levels"])
    b = torch.from_numpy(gmg.random_vector(n, 1)).cuda()
    x0 = gmg.random_vector(n, w["seed_x"])
    x = torch.from_numpy(x0).cuda()
    setup = time.time() - t0
    kw = dict(smoother="jacobi", smoother_omega=1.0, smoothing_omega=0.7, pre_steps=w["pre"], post_steps=w["post"],
              cycle="F", adaptive_correction=True, reduction=reduction)
    gmg.solve_device(prob, b.data_ptr(), x.data_ptr(), gmg.CycleSpec(tolerance=1e-30, max_cycles=2, **kw))  # warm
    x.copy_(torch.from_numpy(x0))
    spec = gmg.CycleSpec(tolerance=1e-30, max_cycles=10, **kw)
    torch.cuda.synchronize()
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    ev0.record()
    rep = gmg.solve_device(prob, b.data_ptr(), x.data_ptr(), spec)
    ev1.record()
    torch.cuda.synchronize()
    ms = ev0.elapsed_time(ev1)
    x.copy_(torch.from_numpy(x0))
    table = per_level_table(gmg.profile_cycle(prob, spec, b.data_ptr(), x.data_ptr(), skip=4), peak, l2_bytes)
    out = {"config": "C5: " + w["desc"] + ", exactly 10 F-cycles (tol 1e-30, max_cycles 10)", "dof": n,
           "cycles": rep.iterations, "ms_per_cycle": ms / rep.iterations,
           "value": n * rep.iterations / (ms / 1e3), "unit": "DOF*cycles/s",
           "residual_first_last": [rep.residual_history[0], rep.residual_history[-1]],
           "host_setup_s": round(setup, 1), "per_level": table,
           "timing": "one gmg_dev_solve_devptr call of 10 cycles, CUDA events on the solver stream (incl. r0 and "
                     "|b| norms)"}
    prob.close()
    del b, x
    torch.cuda.empty_cache()
    return out


def run_ours(args):
    import torch
    ws, rank, local = dist_env()
    if ws > 1:
        os.environ.setdefault("NCCL_DEBUG", "INFO")
        os.environ.setdefault("NCCL_DEBUG_SUBSYS", "INIT")
        os.environ.setdefault("NCCL_DEBUG_FILE", "/dev/stderr")
        import torch.distributed as dist
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    torch.cuda.set_device(local)
    from paper_0805_3041_b200 import gmg

    wl = args.workload
    w = WORKLOADS[wl]
    L = w["levels"]
    pargs = wl_args(w, ws)
    sharded = ws > 1 and args.parallel == "slabs"
    if sharded:
        # one NCCL group for the row slabs; rank 0's unique id travels over the torch group
        ids = [gmg.unique_id() if rank == 0 else None]
        torch.distributed.broadcast_object_list(ids, src=0)
        prob = gmg.MultilevelProblem(*pargs, device=local,
                                     slabs=gmg.Slabs(world=ws, rank=rank, min_rows=255, nccl_id=ids[0]))
        # rank 0 also keeps an unsharded copy for the single-kernel roofline and per-level legs
        single = gmg.MultilevelProblem(*pargs, device=local) if rank == 0 else None
    else:
        prob = gmg.MultilevelProblem(*pargs, device=local)
        single = prob
    n = prob.n(L)
    b_host = gmg.random_vector(n, 1)
    x0_host = np.zeros(n) if not w["seed_x"] else gmg.random_vector(n, w["seed_x"])
    b_dev = torch.from_numpy(b_host).cuda()
    x_dev = torch.from_numpy(x0_host).cuda()
    spec_kw = dict(smoother="jacobi", smoother_omega=1.0, smoothing_omega=0.7, pre_steps=w["pre"],
                   post_steps=w["post"], cycle="F", adaptive_correction=True, reduction=args.reduction)

    def barrier():
        if ws > 1:
            torch.distributed.barrier()
        torch.cuda.synchronize()

    # warm-up: W cycles (captures the CUDA graphs)
    gmg.solve_device(prob, b_dev.data_ptr(), x_dev.data_ptr(),
                     gmg.CycleSpec(tolerance=1e-300, max_cycles=max(1, args.warmup), **spec_kw))
    x_dev.copy_(torch.from_numpy(x0_host))
    spec = gmg.CycleSpec(tolerance=1e-300, max_cycles=args.steps, **spec_kw)

    barrier()
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with ClockSampler(local) as clk:
        ev0.record()
        rep = gmg.solve_device(prob, b_dev.data_ptr(), x_dev.data_ptr(), spec)
        ev1.record()
        torch.cuda.synchronize()
    ms = ev0.elapsed_time(ev1)
    barrier()
    t = torch.tensor([ms], device="cuda")
    if ws > 1:
        torch.distributed.all_reduce(t, op=torch.distributed.ReduceOp.MAX)
    ms_max = float(t.item())
    jobs = 1 if sharded else ws  # grids solved by the whole job
    value = jobs * n * args.steps / (ms_max / 1e3)

    peak, peak_src = load_peaks()
    l2_bytes = torch.cuda.get_device_properties(local).L2_cache_size
    roof, per_level, per_cycle = None, None, None
    if rank == 0:
        # roofline: the finest post-smoother, timed live (CUDA events on the solver stream)
        ms_k, bytes_k = gmg.time_smoother(single, spec, variant=1, reps=20)
        achieved = bytes_k / (ms_k / 1e3) / 1e9
        ms_pre, bytes_pre = gmg.time_smoother(single, spec, variant=0, reps=20)
        traffic = None
        tfile = os.path.join(ROOT, "profiles", "traffic.json")
        if os.path.exists(tfile):
            try:
                traffic = json.load(open(tfile)).get(f"{wl}/post_smoother")
            except Exception:
                traffic = None
        roof = {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s", "frac": achieved / peak,
                "traffic": traffic,
                "traffic_source": "profile constant: dram__bytes_read.sum + dram__bytes_write.sum of this kernel "
                                  "from the committed ncu --set full capture (profiles/traffic.json); not measured "
                                  "in this run",
                "kernel": "k_smooth4<2,CORRECT> finest post-smoother (u+omega*P uc, 2 Jacobi steps fused)",
                "bytes_per_launch": bytes_k, "ms_per_launch": ms_k, "peak_source": peak_src,
                "pre_smoother_GBps": bytes_pre / (ms_pre / 1e3) / 1e9}
        per_cycle = gmg.cycle_kernel_count(single, spec)
        if ws == 1 and not args.no_per_level:
            x_dev.copy_(torch.from_numpy(x0_host))
            # cycle 5 of the solve (mid-convergence; a cycle's exact-sum records depend on the data)
            per_level = per_level_table(gmg.profile_cycle(single, spec, b_dev.data_ptr(), x_dev.data_ptr(), skip=4),
                                        peak, l2_bytes)
    if ws > 1:
        barrier()

    # e2e: public C-ABI solve with pinned host buffers, to the reference tolerance
    pin_b = torch.from_numpy(b_host).pin_memory()
    pin_x = torch.zeros(n, dtype=torch.float64).pin_memory()
    e2e_spec = gmg.CycleSpec(tolerance=w["tol"] if w["tol"] > 1e-29 else 1e-300,
                             max_cycles=args.steps if w["tol"] <= 1e-29 else 50, **spec_kw)
    e2e_cycles, e2e_time = 0, 0.0
    e2e_steps = max(1, min(args.e2e_steps, args.steps))
    for _ in range(e2e_steps):
        xnp = pin_x.numpy()
        xnp[:] = x0_host
        barrier()
        t0 = time.perf_counter()
        r = gmg.solve(prob, pin_b.numpy(), e2e_spec, xnp)
        torch.cuda.synchronize()
        e2e_time += time.perf_counter() - t0
        e2e_cycles += r.iterations
    et = torch.tensor([e2e_time], device="cuda", dtype=torch.float64)
    if ws > 1:
        torch.distributed.all_reduce(et, op=torch.distributed.ReduceOp.MAX)
    e2e_value = jobs * n * e2e_cycles / float(et.item())
    # the drop-in C++ shim passes pageable std::vector memory: the same call on pageable buffers
    e2e_pageable = None
    if rank == 0 and ws == 1:
        for _ in range(2):  # the first call allocates the library's pinned staging ring: warm-up
            xp = x0_host.copy()
            t0 = time.perf_counter()
            r = gmg.solve(prob, b_host, e2e_spec, xp)
            e2e_pageable = n * r.iterations / (time.perf_counter() - t0)
    del pin_b, pin_x

    c5 = None
    if rank == 0 and ws == 1 and wl == "C4" and not args.no_c5:
        if single is not prob:
            single.close()
        c5 = run_c5(gmg, torch, peak, l2_bytes, args.reduction)

    cpu = None
    if rank == 0 and ws == 1 and not args.no_cpu_baseline:
        v, info = cpu_reference_fcycle(wl, threads=1, cycles=1)
        cpu = {"value": v, "unit": "DOF*cycles/s", "cores": 1, "kind": info["kind"], "host": host_info(),
               "pinned_cpu": info["pinned_cpus"][0],
               "sample": f"1 F-cycle of {wl} (gmg::solve max_cycles=1 incl. r0/|b| norms) on 1 host core "
                         f"(thread pinned with sched_setaffinity); {info['seconds']} s timed, setup "
                         f"{info['setup_s']} s excluded"}

    if rank == 0:
        hist = rep.residual_history
        info = prob.dist_info()
        line = {
            "metric": "fine-grid DOF*F-cycles/s (fp64)", "value": value, "unit": "DOF*cycles/s",
            "n_gpus": ws, "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms_max / args.steps,
            "higher_is_better": True, "scaling": "strong" if sharded and not w.get("cny_per_rank") else "weak",
            "vs_baseline": None,
            "dtype": "f64",
            "data": "synthetic (seeded U[-1,1] rhs from std::mt19937, as the reference tests)",
            "config": common_config(wl, n),
            "parallelism": (f"row slabs over {ws} GPUs (levels >= {info[2]} sharded, NCCL halos + rank-ordered "
                            f"exact reductions; NCCL communicator of {info[1]} ranks)") if sharded
            else ("replicas" if ws > 1 else "single GPU"),
            "cycles_timed": args.steps, "residual_first_last": [hist[0], hist[-1]],
            "roofline": roof,
            "per_level": per_level,
            "c5": c5,
            "cpu_baseline": cpu,
            "e2e": {"value": e2e_value, "unit": "DOF*cycles/s", "h2d_bytes_per_step": 2 * n * 8,
                    "d2h_bytes_per_step": n * 8 + 8 * 51, "cycles_per_step": e2e_cycles / e2e_steps,
                    "pageable_value": e2e_pageable,
                    "note": "gmg_dev_solve on pinned host buffers to the reference tolerance (pageable_value: the "
                            "same call on pageable numpy buffers, as the C++ shim passes std::vector memory; staged "
                            "through the library's pinned ring by host threads, second call)"},
            "gpu_launches": (per_cycle or 0) * args.steps + 9,
            "clocks": clk.summary(),
        }
        print(json.dumps(line), flush=True)
    if ws > 1:
        torch.distributed.destroy_process_group()


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=None)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", choices=["ours", "reference"], default="ours")
    ap.add_argument("--workload", choices=sorted(WORKLOADS), default="C4")
    ap.add_argument("--reduction", choices=["exact", "fast"], default="exact")
    ap.add_argument("--e2e-steps", type=int, default=2)
    ap.add_argument("--ref-threads", type=int, default=0)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--parallel", choices=["slabs", "replicas"], default="slabs")
    ap.add_argument("--no-c5", action="store_true", help="skip the C5 (config 5) sub-measurement")
    ap.add_argument("--no-per-level", action="store_true")
    args = ap.parse_args()
    maybe_spawn(args)
    if args.warmup < 3:
        args.warmup = 3
    if args.impl == "reference":
        run_reference_arm(args)
    else:
        run_ours(args)


if __name__ == "__main__":
    main()
