"""Python mirror of the reference gmg2d solver API over the C ABI (include/gmg_b200.h).

Names, argument meaning and error behaviour follow the reference's free
functions in namespace gmg (/root/reference/proj/include/gmg/*.hpp):

    build a problem   MultilevelProblem(levels, coarse_nx, coarse_ny, grading, coords, alpha, beta)
                        <- build_hierarchy (mesh.hpp:70-71) + MultilevelProblem (cycle.hpp:62-78)
    solve             solve(prob, b, spec, x) -> SolveReport   (cycle.hpp:101-106)
    one cycle         mg_cycle(prob, level, u0, g, spec)       (cycle.hpp:89-94)
    operators         apply, residual (stencil.hpp:41-47), smooth_step (smoother.hpp:77-78),
                      restriction, prolongation (transfer.hpp:12-17), adaptive_omega
                      (cycle.hpp:84-87), coarse_solve (BandedCholesky::solve, stencil.hpp:54),
                      norm_l2, dot, axpy (grid_function.hpp:29-34)

Grid functions are float64 numpy arrays of nx*ny interior values, row-major
with x fastest (GridFunction::v). Every computation runs on the GPU through
libgmg_b200.so; there is no CPU fallback — importing this module on a machine
without the built library raises, and calls without a GPU return GMG_ERR_CUDA.

Exceptions mirror the reference: std::logic_error -> LogicError,
std::invalid_argument -> InvalidArgument (a ValueError), std::runtime_error ->
GmgRuntimeError, gmg::DivergenceError -> DivergenceError (carries .report).
"""
from __future__ import annotations

import ctypes as C
import os
from dataclasses import dataclass, field
from typing import List, Optional

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("GMG_LIB_PATH") or os.path.join(_HERE, "libgmg_b200.so")  # override: A/B of alternative builds

GMG_OK, GMG_ERR_LOGIC, GMG_ERR_INVALID, GMG_ERR_RUNTIME, GMG_DIVERGED, GMG_ERR_CUDA, \
    GMG_ERR_UNSUPPORTED = range(7)

SMOOTHERS = ["richardson", "jacobi", "gauss_seidel", "sor", "ilu0", "tri_x", "tri_y", "adi",
             "gstri_x", "gstri_y", "gsadi"]
CYCLES = {"V": 0, "W": 1, "F": 2}
COORDS = {"cartesian": 0, "cylindrical": 1, "spherical": 2, "polar": 3}  # polar: BASELINE C3, no reference
REDUCTIONS = {"exact": 0, "fast": 1}
UNLIMITED = (1 << 64) - 1

# The C-ABI symbols include/gmg_b200.h declares (checked by tests/test_cabi.py).
EXPORTS = [
    "gmg_last_error", "gmg_version", "gmg_dev_problem_create", "gmg_dev_problem_destroy",
    "gmg_dev_num_levels", "gmg_dev_level_shape", "gmg_dev_level_coef_kind", "gmg_dev_solve",
    "gmg_dev_solve_devptr", "gmg_dev_mg_cycle", "gmg_dev_apply", "gmg_dev_residual",
    "gmg_dev_smooth_step", "gmg_dev_restriction", "gmg_dev_prolongation", "gmg_dev_adaptive_omega",
    "gmg_dev_coarse_solve", "gmg_dev_norm_l2", "gmg_dev_dot", "gmg_dev_axpy",
    "gmg_dev_time_smoother", "gmg_dev_cycle_kernel_count", "gmg_dev_seqsum_stats", "gmg_host_problem_create",
    "gmg_host_random_vector", "gmg_host_seqsum_emulate", "gmg_dev_problem_create_slabs", "gmg_dist_unique_id",
    "gmg_dev_dist_info", "gmg_dev_level_window", "gmg_host_problem_create_slabs", "gmg_host_slab_plan",
    "gmg_dev_make_start_vector", "gmg_dev_profile_cycle",
]
START_KINDS = ["zero", "nested", "continuation"]  # gmg::StartVectorKind (config.hpp:11)


class GmgError(Exception):
    code = -1


class LogicError(GmgError):
    code = GMG_ERR_LOGIC


class InvalidArgument(GmgError, ValueError):
    code = GMG_ERR_INVALID


class GmgRuntimeError(GmgError, RuntimeError):
    code = GMG_ERR_RUNTIME


class DivergenceError(GmgRuntimeError):
    code = GMG_DIVERGED

    def __init__(self, msg, report):
        super().__init__(msg)
        self.report = report


class CudaError(GmgError, RuntimeError):
    code = GMG_ERR_CUDA


class Unsupported(GmgError, NotImplementedError):
    code = GMG_ERR_UNSUPPORTED


_EXC = {GMG_ERR_LOGIC: LogicError, GMG_ERR_INVALID: InvalidArgument,
        GMG_ERR_RUNTIME: GmgRuntimeError, GMG_ERR_CUDA: CudaError,
        GMG_ERR_UNSUPPORTED: Unsupported}

_dp = C.POINTER(C.c_double)


class _LevelDesc(C.Structure):
    _fields_ = [("level", C.c_int), ("nx", C.c_int), ("ny", C.c_int), ("x", _dp), ("y", _dp),
                ("c", _dp), ("n", _dp), ("s", _dp), ("e", _dp), ("w", _dp)]


class _ProblemDesc(C.Structure):
    _fields_ = [("num_levels", C.c_int), ("levels", C.POINTER(_LevelDesc)), ("device", C.c_int),
                ("periodic_y", C.c_int), ("alpha", C.c_double), ("beta", C.c_double), ("coords", C.c_int)]


class _SlabDesc(C.Structure):
    _fields_ = [("world", C.c_int), ("rank", C.c_int), ("min_rows", C.c_int), ("nccl_id", C.c_void_p)]


class _CycleDesc(C.Structure):
    _fields_ = [("cycle", C.c_int), ("pre_steps", C.c_int), ("post_steps", C.c_int),
                ("adaptive_correction", C.c_int), ("correction_omega", C.c_double),
                ("smoother_kind", C.c_int), ("smoother_omega", C.c_double),
                ("smoothing_omega", C.c_double), ("tolerance", C.c_double),
                ("max_cycles", C.c_int), ("coarse_direct_max_neq", C.c_ulonglong),
                ("reduction", C.c_int)]


class _ProfEntry(C.Structure):
    _fields_ = [("kernel", C.c_char * 48), ("level", C.c_int), ("bytes", C.c_double), ("ms", C.c_double)]


class _Report(C.Structure):
    _fields_ = [("iterations", C.c_int), ("converged", C.c_int), ("wall_seconds", C.c_double),
                ("residual_history", _dp), ("convergence_factors", _dp), ("history_len", C.c_int),
                ("message", C.c_char * 256)]


_lib = None


def lib() -> C.CDLL:
    """Loads libgmg_b200.so (fails loudly if it was not built)."""
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise ImportError(f"{LIB_PATH} not built: run `python -m paper_0805_3041_b200.build`")
        L = C.CDLL(LIB_PATH)
        L.gmg_last_error.restype = C.c_char_p
        L.gmg_version.restype = C.c_char_p
        L.gmg_dev_problem_create.argtypes = [C.POINTER(_ProblemDesc), C.POINTER(C.c_void_p)]
        L.gmg_dev_problem_destroy.argtypes = [C.c_void_p]
        L.gmg_dev_num_levels.argtypes = [C.c_void_p]
        L.gmg_dev_level_shape.argtypes = [C.c_void_p, C.c_int, C.POINTER(C.c_int), C.POINTER(C.c_int)]
        L.gmg_dev_level_coef_kind.argtypes = [C.c_void_p, C.c_int]
        L.gmg_dev_solve.argtypes = [C.c_void_p, C.POINTER(_CycleDesc), _dp, _dp, C.POINTER(_Report)]
        L.gmg_dev_solve_devptr.argtypes = [C.c_void_p, C.POINTER(_CycleDesc), C.c_void_p, C.c_void_p,
                                           C.POINTER(_Report)]
        L.gmg_dev_mg_cycle.argtypes = [C.c_void_p, C.POINTER(_CycleDesc), C.c_int, _dp, _dp, _dp]
        L.gmg_dev_apply.argtypes = [C.c_void_p, C.c_int, _dp, _dp]
        L.gmg_dev_make_start_vector.argtypes = [C.c_void_p, C.POINTER(_CycleDesc), C.c_int, _dp, _dp]
        L.gmg_dev_residual.argtypes = [C.c_void_p, C.c_int, _dp, _dp, _dp]
        L.gmg_dev_smooth_step.argtypes = [C.c_void_p, C.c_int, C.c_int, C.c_double, C.c_double, _dp, _dp, _dp]
        L.gmg_dev_restriction.argtypes = [C.c_void_p, C.c_int, _dp, _dp]
        L.gmg_dev_prolongation.argtypes = [C.c_void_p, C.c_int, _dp, _dp]
        L.gmg_dev_adaptive_omega.argtypes = [C.c_void_p, C.c_int, _dp, _dp, _dp]
        L.gmg_dev_coarse_solve.argtypes = [C.c_void_p, _dp, _dp]
        L.gmg_dev_norm_l2.argtypes = [C.c_void_p, C.c_longlong, _dp, C.c_int, _dp]
        L.gmg_dev_dot.argtypes = [C.c_void_p, C.c_longlong, _dp, _dp, C.c_int, _dp]
        L.gmg_dev_axpy.argtypes = [C.c_void_p, C.c_longlong, C.c_double, _dp, _dp]
        L.gmg_dev_time_smoother.argtypes = [C.c_void_p, C.POINTER(_CycleDesc), C.c_int, C.c_int, _dp, _dp]
        L.gmg_dev_seqsum_stats.argtypes = [C.c_void_p, C.c_int, C.POINTER(C.c_ulonglong)]
        L.gmg_dev_profile_cycle.argtypes = [C.c_void_p, C.POINTER(_CycleDesc), C.c_void_p, C.c_void_p, C.c_int,
                                            C.c_int, C.POINTER(_ProfEntry), C.POINTER(C.c_int)]
        L.gmg_dev_cycle_kernel_count.argtypes = [C.c_void_p, C.POINTER(_CycleDesc), C.POINTER(C.c_int)]
        L.gmg_host_problem_create.argtypes = [C.c_int, C.c_int, C.c_int, C.c_double, C.c_double,
                                              C.c_int, C.c_double, C.c_double, C.c_int,
                                              C.POINTER(C.c_void_p)]
        L.gmg_host_random_vector.argtypes = [C.c_longlong, C.c_uint, _dp]
        L.gmg_dev_problem_create_slabs.argtypes = [C.POINTER(_ProblemDesc), C.POINTER(_SlabDesc),
                                                   C.POINTER(C.c_void_p)]
        L.gmg_dist_unique_id.argtypes = [C.c_char_p]
        L.gmg_dev_dist_info.argtypes = [C.c_void_p, C.POINTER(C.c_int), C.POINTER(C.c_int), C.POINTER(C.c_int)]
        L.gmg_dev_level_window.argtypes = [C.c_void_p, C.c_int, C.POINTER(C.c_int), C.POINTER(C.c_int)]
        L.gmg_host_problem_create_slabs.argtypes = [C.c_int, C.c_int, C.c_int, C.c_double, C.c_double,
                                                    C.c_int, C.c_double, C.c_double, C.c_int,
                                                    C.POINTER(_SlabDesc), C.POINTER(C.c_void_p)]
        L.gmg_host_slab_plan.argtypes = [C.c_int, C.POINTER(C.c_int), C.c_int, C.c_int, C.c_int,
                                         C.POINTER(C.c_int), C.POINTER(C.c_int), C.POINTER(C.c_int)]
        L.gmg_host_seqsum_emulate.argtypes = [C.c_longlong, _dp, C.c_int, C.c_int, _dp,
                                              C.POINTER(C.c_longlong)]
        _lib = L
    return _lib


def _check(code: int):
    if code != GMG_OK:
        msg = lib().gmg_last_error().decode()
        raise _EXC.get(code, GmgError)(msg)


def _arr(a, n=None) -> np.ndarray:
    a = np.ascontiguousarray(a, dtype=np.float64)
    if n is not None and a.size != n:
        raise LogicError(f"grid function has {a.size} values, level expects {n}")
    return a


def _p(a: np.ndarray):
    return a.ctypes.data_as(_dp)


@dataclass
class Slabs:
    """Row-slab distribution of a problem (gmg_slab_desc): rank=None puts all `world`
    slabs in this process on one GPU (virtual ranks); rank>=0 is this process's slab
    of an NCCL group whose id (bytes from unique_id() on rank 0) is shared by the caller."""
    world: int
    rank: Optional[int] = None
    min_rows: int = 255
    nccl_id: Optional[bytes] = None

    def _c(self):
        buf = C.create_string_buffer(self.nccl_id, 128) if self.nccl_id is not None else None
        sd = _SlabDesc(self.world, -1 if self.rank is None else self.rank, self.min_rows,
                       C.cast(buf, C.c_void_p) if buf is not None else None)
        return sd, buf


def unique_id() -> bytes:
    """ncclGetUniqueId (rank 0 of a row-slab group)."""
    buf = C.create_string_buffer(128)
    _check(lib().gmg_dist_unique_id(buf))
    return buf.raw


def slab_plan(ny, world: int, min_rows: int = 255, halo: int = 4):
    """The row-slab partition (host only): (first sharded level, w0[level][rank], w1[level][rank])."""
    L = len(ny)
    nya = (C.c_int * L)(*ny)
    w0 = (C.c_int * (L * world))()
    w1 = (C.c_int * (L * world))()
    first = C.c_int()
    _check(lib().gmg_host_slab_plan(L, nya, world, min_rows, halo, C.byref(first), w0, w1))
    return (first.value, [[w0[l * world + r] for r in range(world)] for l in range(L)],
            [[w1[l * world + r] for r in range(world)] for l in range(L)])


@dataclass
class CycleSpec:
    """gmg::CycleSpec (cycle.hpp:23-39) with SmootherSpec folded in; defaults as the reference."""
    cycle: str = "F"
    pre_steps: int = 2
    post_steps: int = 2
    adaptive_correction: bool = True
    correction_omega: float = 1.0
    smoother: str = "gauss_seidel"
    smoother_omega: float = 1.0
    smoothing_omega: float = 0.7
    tolerance: float = 1e-4
    max_cycles: int = 50
    coarse_direct_max_neq: int = UNLIMITED
    reduction: str = "exact"

    def _c(self) -> _CycleDesc:
        if self.cycle not in CYCLES:
            raise InvalidArgument("cycle: must be one of V, W, F")
        if self.smoother not in SMOOTHERS:
            raise InvalidArgument(f"smoother: unknown kind '{self.smoother}'")
        return _CycleDesc(CYCLES[self.cycle], self.pre_steps, self.post_steps,
                          int(bool(self.adaptive_correction)), float(self.correction_omega),
                          SMOOTHERS.index(self.smoother), float(self.smoother_omega),
                          float(self.smoothing_omega), float(self.tolerance), int(self.max_cycles),
                          int(self.coarse_direct_max_neq), REDUCTIONS[self.reduction])


@dataclass
class SolveReport:
    """gmg::SolveReport (cycle.hpp:41-47)."""
    iterations: int = 0
    residual_history: List[float] = field(default_factory=list)
    convergence_factors: List[float] = field(default_factory=list)
    converged: bool = False
    wall_seconds: float = 0.0


class MultilevelProblem:
    """Device-resident operators of every level plus the level-1 factorization."""

    def __init__(self, levels: int, coarse_nx: int = 1, coarse_ny: int = 1, grading=(1.0, 1.0),
                 coords: str = "cartesian", alpha: float = 1.0, beta: float = 1.0, device: int = 0,
                 slabs: Optional["Slabs"] = None):
        h = C.c_void_p()
        if coords not in COORDS:
            raise InvalidArgument(f"coords: unknown coordinate system '{coords}'")
        args = (levels, coarse_nx, coarse_ny, float(grading[0]), float(grading[1]), COORDS[coords], float(alpha),
                float(beta), device)
        if slabs is None:
            _check(lib().gmg_host_problem_create(*args, C.byref(h)))
        else:
            sd, _keep = slabs._c()
            _check(lib().gmg_host_problem_create_slabs(*args, C.byref(sd), C.byref(h)))
        self._init(h)

    @classmethod
    def from_levels(cls, levels: list, device: int = 0) -> "MultilevelProblem":
        """levels[l-1] = dict(nx, ny, x, y, c, n, s, e, w) — a reference MultilevelProblem's data."""
        keep = []
        descs = (_LevelDesc * len(levels))()
        for q, L in enumerate(levels):
            arrs = {k: _arr(L[k]) for k in ("x", "y", "c", "n", "s", "e", "w")}
            keep.append(arrs)
            descs[q] = _LevelDesc(q + 1, L["nx"], L["ny"], *[_p(arrs[k]) for k in ("x", "y", "c", "n", "s", "e", "w")])
        pd = _ProblemDesc(len(levels), descs, device, 0, 0.0, 0.0, 0)  # no physics: arrays as given
        h = C.c_void_p()
        _check(lib().gmg_dev_problem_create(C.byref(pd), C.byref(h)))
        obj = cls.__new__(cls)
        obj._init(h)
        return obj

    def _init(self, h):
        self._h = h
        self.num_levels = lib().gmg_dev_num_levels(h)
        self.shapes = {}
        for l in range(1, self.num_levels + 1):
            nx, ny = C.c_int(), C.c_int()
            _check(lib().gmg_dev_level_shape(h, l, C.byref(nx), C.byref(ny)))
            self.shapes[l] = (nx.value, ny.value)

    def n(self, level: int) -> int:
        nx, ny = self.shapes[level]
        return nx * ny

    def dist_info(self):
        """(rank, world, first sharded level) of a row-slab handle; (0, 1, L+1) otherwise."""
        r, w, f = C.c_int(), C.c_int(), C.c_int()
        _check(lib().gmg_dev_dist_info(self._h, C.byref(r), C.byref(w), C.byref(f)))
        return r.value, w.value, f.value

    def level_window(self, level: int):
        a, b = C.c_int(), C.c_int()
        _check(lib().gmg_dev_level_window(self._h, level, C.byref(a), C.byref(b)))
        return a.value, b.value

    def coef_kind(self, level: int) -> str:
        return {0: "const", 1: "rowx", 2: "field", 3: "axes"}.get(lib().gmg_dev_level_coef_kind(self._h, level), "?")

    def close(self):
        if getattr(self, "_h", None):
            lib().gmg_dev_problem_destroy(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


def _report(max_cycles: int):
    hist = np.zeros(max(1, max_cycles) + 1)
    fac = np.zeros(max(1, max_cycles))
    rep = _Report(0, 0, 0.0, _p(hist), _p(fac), 0, b"")
    return rep, hist, fac


def _to_report(rep, hist, fac) -> SolveReport:
    n = rep.history_len
    return SolveReport(rep.iterations, hist[:n].tolist(), fac[: max(0, n - 1)].tolist(),
                       bool(rep.converged), rep.wall_seconds)


def solve(prob: MultilevelProblem, b, spec: CycleSpec, x: np.ndarray) -> SolveReport:
    """gmg::solve: x (float64 array, start vector) is overwritten with the solution."""
    L = prob.num_levels
    b = _arr(b, prob.n(L))
    if not (isinstance(x, np.ndarray) and x.dtype == np.float64 and x.flags.c_contiguous and x.size == prob.n(L)):
        raise LogicError("solve: x must be a contiguous float64 array of the finest level")
    rep, hist, fac = _report(spec.max_cycles)
    code = lib().gmg_dev_solve(prob._h, C.byref(spec._c()), _p(b), _p(x), C.byref(rep))
    if code == GMG_DIVERGED:
        raise DivergenceError(lib().gmg_last_error().decode(), _to_report(rep, hist, fac))
    _check(code)
    return _to_report(rep, hist, fac)


def solve_device(prob: MultilevelProblem, b_ptr: int, x_ptr: int, spec: CycleSpec) -> SolveReport:
    """gmg::solve with b and x already in device memory (raw CUDA pointers, reference layout)."""
    rep, hist, fac = _report(spec.max_cycles)
    code = lib().gmg_dev_solve_devptr(prob._h, C.byref(spec._c()), C.c_void_p(b_ptr), C.c_void_p(x_ptr),
                                      C.byref(rep))
    if code == GMG_DIVERGED:
        raise DivergenceError(lib().gmg_last_error().decode(), _to_report(rep, hist, fac))
    _check(code)
    return _to_report(rep, hist, fac)


def mg_cycle(prob: MultilevelProblem, level: int, u0, g, spec: CycleSpec) -> np.ndarray:
    u0 = _arr(u0, prob.n(level))
    g = _arr(g, prob.n(level))
    u = np.zeros(prob.n(level))
    _check(lib().gmg_dev_mg_cycle(prob._h, C.byref(spec._c()), level, _p(u0), _p(g), _p(u)))
    return u


def make_start_vector(kind: str, prob: MultilevelProblem, spec: CycleSpec, b, source=None) -> np.ndarray:
    """gmg::make_start_vector (study.hpp:20-21, study.cpp:40-79) on the device: "zero",
    "nested" (level-1 solve of the restricted b, then prolongation + one smooth_step of
    spec's smoother per level) or "continuation" (a copy of `source`, the solution of
    a related problem with the same finest shape)."""
    L = prob.num_levels
    n = prob.n(L)
    if kind == "continuation":
        if source is None:
            raise InvalidArgument("start: continuation requires a source solution")
        src = _arr(source)
        if src.size != n:
            raise InvalidArgument("start: continuation source shape does not match")
        return src.copy()
    if kind not in START_KINDS:
        raise InvalidArgument(f"start: unknown start vector '{kind}'")
    b = _arr(b, n)
    x = np.zeros(n)
    _check(lib().gmg_dev_make_start_vector(prob._h, C.byref(spec._c()), START_KINDS.index(kind), _p(b), _p(x)))
    return x


def apply(prob: MultilevelProblem, level: int, x) -> np.ndarray:
    x = _arr(x, prob.n(level))
    y = np.zeros_like(x)
    _check(lib().gmg_dev_apply(prob._h, level, _p(x), _p(y)))
    return y


def residual(prob: MultilevelProblem, level: int, x, b) -> np.ndarray:
    x = _arr(x, prob.n(level))
    b = _arr(b, prob.n(level))
    r = np.zeros_like(x)
    _check(lib().gmg_dev_residual(prob._h, level, _p(x), _p(b), _p(r)))
    return r


def smooth_step(prob: MultilevelProblem, level: int, kind: str, smoother_omega: float, x, b,
                omega_damp: float) -> np.ndarray:
    x = _arr(x, prob.n(level))
    b = _arr(b, prob.n(level))
    out = np.zeros_like(x)
    if kind not in SMOOTHERS:
        raise InvalidArgument(f"smoother: unknown kind '{kind}'")
    _check(lib().gmg_dev_smooth_step(prob._h, level, SMOOTHERS.index(kind), float(smoother_omega),
                                     float(omega_damp), _p(x), _p(b), _p(out)))
    return out


def restriction(prob: MultilevelProblem, fine_level: int, fine) -> np.ndarray:
    fine = _arr(fine, prob.n(fine_level))
    out = np.zeros(prob.n(fine_level - 1)) if fine_level >= 2 else np.zeros(1)
    _check(lib().gmg_dev_restriction(prob._h, fine_level, _p(fine), _p(out)))
    return out


def prolongation(prob: MultilevelProblem, coarse_level: int, coarse) -> np.ndarray:
    coarse = _arr(coarse, prob.n(coarse_level))
    out = np.zeros(prob.n(coarse_level + 1)) if coarse_level < prob.num_levels else np.zeros(1)
    _check(lib().gmg_dev_prolongation(prob._h, coarse_level, _p(coarse), _p(out)))
    return out


def adaptive_omega(prob: MultilevelProblem, level: int, defect, correction) -> float:
    d = _arr(defect, prob.n(level))
    c = _arr(correction, prob.n(level))
    w = np.zeros(1)
    _check(lib().gmg_dev_adaptive_omega(prob._h, level, _p(d), _p(c), _p(w)))
    return float(w[0])


def coarse_solve(prob: MultilevelProblem, b) -> np.ndarray:
    b = _arr(b, prob.n(1))
    x = np.zeros_like(b)
    _check(lib().gmg_dev_coarse_solve(prob._h, _p(b), _p(x)))
    return x


def norm_l2(prob: MultilevelProblem, v, reduction: str = "exact") -> float:
    v = _arr(v)
    out = np.zeros(1)
    _check(lib().gmg_dev_norm_l2(prob._h, v.size, _p(v), REDUCTIONS[reduction], _p(out)))
    return float(out[0])


def dot(prob: MultilevelProblem, a, b, reduction: str = "exact") -> float:
    a = _arr(a)
    b = _arr(b, a.size)
    out = np.zeros(1)
    _check(lib().gmg_dev_dot(prob._h, a.size, _p(a), _p(b), REDUCTIONS[reduction], _p(out)))
    return float(out[0])


def axpy(prob: MultilevelProblem, alpha: float, x, y: np.ndarray) -> None:
    x = _arr(x)
    if not (isinstance(y, np.ndarray) and y.dtype == np.float64 and y.flags.c_contiguous and y.size == x.size):
        raise LogicError("axpy: grid functions live on different levels")
    _check(lib().gmg_dev_axpy(prob._h, x.size, float(alpha), _p(x), _p(y)))


def random_vector(n: int, seed: int) -> np.ndarray:
    """std::mt19937(seed) + uniform_real_distribution<double>(-1,1) (tests/oracles.hpp:252-258)."""
    v = np.zeros(n)
    lib().gmg_host_random_vector(n, seed, _p(v))
    return v


def seqsum_emulate(terms, threads: int = 256, ept: int = 32):
    """Host emulation of the device exact-order summation engine (for CPU tests)."""
    t = _arr(terms)
    out = np.zeros(1)
    stats = (C.c_longlong * 4)()
    _check(lib().gmg_host_seqsum_emulate(t.size, _p(t), threads, ept, _p(out), stats))
    return float(out[0]), list(stats)


def time_smoother(prob: MultilevelProblem, spec: CycleSpec, variant: int = 0, reps: int = 20):
    ms, by = np.zeros(1), np.zeros(1)
    _check(lib().gmg_dev_time_smoother(prob._h, C.byref(spec._c()), variant, reps, _p(ms), _p(by)))
    return float(ms[0]), float(by[0])


def profile_cycle(prob: MultilevelProblem, spec: CycleSpec, b_ptr: int, x_ptr: int, skip: int = 0, cap: int = 8192):
    """Cycle skip+1 of a solve from device arrays b, x with CUDA events around every
    launch: list of dicts (kernel, level, bytes = algorithmic bytes, ms)."""
    buf = (_ProfEntry * cap)()
    n = C.c_int()
    _check(lib().gmg_dev_profile_cycle(prob._h, C.byref(spec._c()), C.c_void_p(b_ptr), C.c_void_p(x_ptr), skip, cap,
                                       buf, C.byref(n)))
    return [dict(kernel=buf[k].kernel.decode(), level=buf[k].level, bytes=buf[k].bytes, ms=buf[k].ms)
            for k in range(min(n.value, cap))]


def cycle_kernel_count(prob: MultilevelProblem, spec: CycleSpec) -> int:
    n = C.c_int()
    _check(lib().gmg_dev_cycle_kernel_count(prob._h, C.byref(spec._c()), C.byref(n)))
    return n.value


def seqsum_stats(prob: MultilevelProblem, reset: bool = True) -> dict:
    """Exact-order summation engine counters since the last reset."""
    a = (C.c_ulonglong * 16)()
    _check(lib().gmg_dev_seqsum_stats(prob._h, int(reset), a))
    keys = ["sums", "records", "chain_cycles", "rewalk_cycles", "break_adds", "rewalks",
            "rewalk_terms", "chunks", "walk_load", "walk_prefix_lookback", "walk_thread_walk",
            "walk_block_merge", "walk_run_lookback", "walk_ctas", "dense_chunks", "dense_cycles"]
    return dict(zip(keys, list(a)))
