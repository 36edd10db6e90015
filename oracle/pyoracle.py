"""TEST INFRASTRUCTURE ONLY — ctypes access to the CPU checkers.

Two interchangeable back ends with one method surface:

* ``Oracle`` — the plain-C restatement ``oracle/liboracle.so`` (gmg_oracle.c).
* ``Reference`` — the UNMODIFIED reference library compiled from
  /root/reference/proj/src (``oracle/_ref/libgmg_ref_capi.so``, built by
  oracle/Makefile; the .so travels to the GPU box, the sources do not).

Only tests/, ``__graft_entry__.smoke()`` and bench.py's cpu_baseline/reference
legs import this module, and only as the checker or the timed CPU baseline —
never as the product path.
"""
from __future__ import annotations

import ctypes as C
import os
from dataclasses import dataclass

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ORACLE_SO = os.path.join(HERE, "liboracle.so")
REF_SO = os.path.join(HERE, "_ref", "libgmg_ref_capi.so")

COORDS = {"cartesian": 0, "cylindrical": 1, "spherical": 2, "polar": 3}  # polar: oracle and device only (no reference)
SMOOTHERS = ["richardson", "jacobi", "gauss_seidel", "sor", "ilu0", "tri_x", "tri_y",
             "adi", "gstri_x", "gstri_y", "gsadi"]
CYCLES = {"V": 0, "W": 1, "F": 2}
START_KINDS = ["zero", "nested", "continuation"]  # gmg::StartVectorKind (config.hpp:11)
UNLIMITED = (1 << 64) - 1

_dp = C.POINTER(C.c_double)


def _ptr(a: np.ndarray):
    assert a.dtype == np.float64 and a.flags.c_contiguous
    return a.ctypes.data_as(_dp)


class CheckerError(RuntimeError):
    def __init__(self, code: int, msg: str):
        super().__init__(f"[{code}] {msg}")
        self.code = code
        self.msg = msg


class _Spec(C.Structure):
    _fields_ = [("cycle", C.c_int), ("pre_steps", C.c_int), ("post_steps", C.c_int),
                ("adaptive_correction", C.c_int), ("correction_omega", C.c_double),
                ("smoother_kind", C.c_int), ("smoother_omega", C.c_double),
                ("smoothing_omega", C.c_double), ("tolerance", C.c_double),
                ("max_cycles", C.c_int), ("coarse_direct_max_neq", C.c_ulonglong)]


@dataclass
class CycleSpec:
    """Mirror of gmg::CycleSpec (include/gmg/cycle.hpp:23-39) with its defaults."""
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

    def to_c(self) -> _Spec:
        return _Spec(CYCLES[self.cycle], self.pre_steps, self.post_steps,
                     int(self.adaptive_correction), self.correction_omega,
                     SMOOTHERS.index(self.smoother), self.smoother_omega,
                     self.smoothing_omega, self.tolerance, self.max_cycles,
                     self.coarse_direct_max_neq)


@dataclass
class SolveResult:
    status: int
    history: list
    iterations: int
    converged: bool
    wall_seconds: float
    message: str


class _Backend:
    lib: C.CDLL

    def __init__(self, levels, coarse_nx=1, coarse_ny=1, grading=(1.0, 1.0),
                 coords="cartesian", alpha=1.0, beta=1.0):
        self.levels = levels
        self.handle = self._create(levels, coarse_nx, coarse_ny, float(grading[0]),
                                   float(grading[1]), COORDS[coords], float(alpha), float(beta))
        self.shapes = {}
        for l in range(1, levels + 1):
            nx, ny = C.c_int(), C.c_int()
            self._shape(l, C.byref(nx), C.byref(ny))
            self.shapes[l] = (nx.value, ny.value)

    # sizes ---------------------------------------------------------------
    def n(self, level):
        nx, ny = self.shapes[level]
        return nx * ny

    def coords(self, level):
        nx, ny = self.shapes[level]
        x = np.zeros(nx + 2)
        y = np.zeros(ny + 2)
        self.lib_call("level_coords", level, _ptr(x), _ptr(y))
        return x, y

    def operator(self, level):
        arrs = [np.zeros(self.n(level)) for _ in range(5)]
        self.lib_call("operator", level, *[_ptr(a) for a in arrs])
        return dict(zip("cnsew", arrs))

    # ops -------------------------------------------------------------------
    def apply(self, level, x):
        y = np.zeros(self.n(level))
        self.lib_call("apply", level, _ptr(np.ascontiguousarray(x, np.float64)), _ptr(y))
        return y

    def residual(self, level, x, b):
        r = np.zeros(self.n(level))
        self.lib_call("residual", level, _ptr(np.ascontiguousarray(x, np.float64)),
                      _ptr(np.ascontiguousarray(b, np.float64)), _ptr(r))
        return r

    def restriction(self, fine_level, f):
        c = np.zeros(self.n(fine_level - 1))
        self.lib_call("restriction", fine_level, _ptr(np.ascontiguousarray(f, np.float64)), _ptr(c))
        return c

    def prolongation(self, coarse_level, c):
        f = np.zeros(self.n(coarse_level + 1))
        self.lib_call("prolongation", coarse_level, _ptr(np.ascontiguousarray(c, np.float64)), _ptr(f))
        return f

    def coarse_solve(self, b):
        x = np.zeros(self.n(1))
        self.lib_call("coarse_solve", _ptr(np.ascontiguousarray(b, np.float64)), _ptr(x))
        return x


class Oracle(_Backend):
    """The C restatement (oracle/gmg_oracle.c)."""

    _lib = None

    @classmethod
    def load(cls):
        if cls._lib is None:
            if not os.path.exists(ORACLE_SO):
                raise FileNotFoundError(f"{ORACLE_SO} missing: run make -C oracle")
            lib = C.CDLL(ORACLE_SO)
            lib.orc_problem_create.restype = C.c_void_p
            lib.orc_problem_create.argtypes = [C.c_int, C.c_int, C.c_int, C.c_double, C.c_double,
                                               C.c_int, C.c_double, C.c_double]
            lib.orc_last_error.restype = C.c_char_p
            lib.orc_norm_l2.restype = C.c_double
            lib.orc_norm_l2.argtypes = [C.c_longlong, _dp]
            lib.orc_dot.restype = C.c_double
            lib.orc_dot.argtypes = [C.c_longlong, _dp, _dp]
            lib.orc_random_vector.argtypes = [C.c_longlong, C.c_uint, _dp]
            lib.orc_smooth_step.argtypes = [C.c_void_p, C.c_int, C.c_int, C.c_double, C.c_double,
                                            _dp, _dp, _dp]
            lib.orc_adaptive_omega.argtypes = [C.c_void_p, C.c_int, _dp, _dp, _dp]
            cls._lib = lib
        return cls._lib

    def __init__(self, *a, **k):
        self.lib = self.load()
        super().__init__(*a, **k)

    def _create(self, *args):
        h = self.lib.orc_problem_create(*args)
        if not h:
            raise CheckerError(2, self.lib.orc_last_error().decode())
        return C.c_void_p(h)

    def _shape(self, l, nx, ny):
        self.lib.orc_level_shape(self.handle, l, nx, ny)

    def lib_call(self, name, *args):
        st = getattr(self.lib, "orc_" + name)(self.handle, *args)
        if st:
            raise CheckerError(st, self.lib.orc_last_error().decode())
        return st

    def __del__(self):
        if getattr(self, "handle", None):
            self.lib.orc_problem_destroy(self.handle)
            self.handle = None

    def smooth_step(self, level, kind, smoother_omega, omega_damp, x, b):
        out = np.zeros(self.n(level))
        self.lib_call("smooth_step", level, SMOOTHERS.index(kind), smoother_omega, omega_damp,
                      _ptr(np.ascontiguousarray(x, np.float64)),
                      _ptr(np.ascontiguousarray(b, np.float64)), _ptr(out))
        return out

    def adaptive_omega(self, level, d, corr):
        w = np.zeros(1)
        self.lib_call("adaptive_omega", level, _ptr(np.ascontiguousarray(d, np.float64)),
                      _ptr(np.ascontiguousarray(corr, np.float64)), _ptr(w))
        return float(w[0])

    def norm_l2(self, v):
        v = np.ascontiguousarray(v, np.float64)
        return self.lib.orc_norm_l2(v.size, _ptr(v))

    def dot(self, a, b):
        a = np.ascontiguousarray(a, np.float64)
        b = np.ascontiguousarray(b, np.float64)
        return self.lib.orc_dot(a.size, _ptr(a), _ptr(b))

    def mg_cycle(self, spec: CycleSpec, level, u0, g):
        u = np.zeros(self.n(level))
        cs = spec.to_c()
        self.lib_call("mg_cycle", C.byref(cs), level, _ptr(np.ascontiguousarray(u0, np.float64)),
                      _ptr(np.ascontiguousarray(g, np.float64)), _ptr(u))
        return u

    def solve(self, spec: CycleSpec, b, x):
        """Runs the oracle solve; x (float64 array) is updated in place."""
        hist = np.zeros(spec.max_cycles + 1)
        hl, it, cv = C.c_int(), C.c_int(), C.c_int()
        cs = spec.to_c()
        st = self.lib.orc_solve(self.handle, C.byref(cs), _ptr(np.ascontiguousarray(b, np.float64)),
                                _ptr(x), _ptr(hist), C.byref(hl), C.byref(it), C.byref(cv))
        msg = self.lib.orc_last_error().decode() if st else ""
        return SolveResult(st, hist[: hl.value].tolist(), it.value, bool(cv.value), 0.0, msg)

    def start_vector(self, spec: CycleSpec, kind, b):
        """make_start_vector (study.cpp:40-79); kind "zero" or "nested"."""
        x = np.zeros(self.n(self.levels))
        cs = spec.to_c()
        self.lib_call("start_vector", C.byref(cs), START_KINDS.index(kind),
                      _ptr(np.ascontiguousarray(b, np.float64)), _ptr(x))
        return x

    @classmethod
    def random_vector(cls, n, seed):
        v = np.zeros(n)
        cls.load().orc_random_vector(n, seed, _ptr(v))
        return v


class Reference(_Backend):
    """The reference library itself, compiled from /root/reference sources."""

    _lib = None

    @staticmethod
    def available() -> bool:
        return os.path.exists(REF_SO)

    @classmethod
    def load(cls):
        if cls._lib is None:
            if not os.path.exists(REF_SO):
                raise FileNotFoundError(f"{REF_SO} missing: run make -C oracle where /root/reference exists")
            lib = C.CDLL(REF_SO)
            lib.ref_problem_create.restype = C.c_void_p
            lib.ref_problem_create.argtypes = [C.c_int, C.c_int, C.c_int, C.c_double, C.c_double,
                                               C.c_int, C.c_double, C.c_double, C.c_char_p, C.c_int]
            lib.ref_problem_destroy.argtypes = [C.c_void_p]
            for name in ("level_shape", "level_coords", "operator", "apply", "residual",
                         "restriction", "prolongation", "coarse_solve"):
                getattr(lib, "ref_" + name).argtypes = None
            lib.ref_norm_l2.restype = C.c_double
            lib.ref_dot.restype = C.c_double
            lib.ref_random_vector.argtypes = [C.c_longlong, C.c_uint, _dp]
            lib.ref_smooth_step.argtypes = [C.c_void_p, C.c_int, C.c_int, C.c_double, C.c_double,
                                            _dp, _dp, _dp, C.c_char_p, C.c_int]
            lib.ref_adaptive_omega.argtypes = [C.c_void_p, C.c_int, _dp, _dp, _dp, C.c_char_p, C.c_int]
            lib.ref_mg_cycle.argtypes = [C.c_void_p, C.c_void_p, C.c_int, _dp, _dp, _dp,
                                         C.c_char_p, C.c_int]
            lib.ref_solve.argtypes = [C.c_void_p, C.c_void_p, _dp, _dp, _dp, C.c_void_p, C.c_void_p,
                                      C.c_void_p, _dp, C.c_char_p, C.c_int]
            cls._lib = lib
        return cls._lib

    def __init__(self, *a, **k):
        self.lib = self.load()
        super().__init__(*a, **k)

    def _create(self, *args):
        err = C.create_string_buffer(256)
        h = self.lib.ref_problem_create(*args, err, 256)
        if not h:
            raise CheckerError(2, err.value.decode())
        return C.c_void_p(h)

    def _shape(self, l, nx, ny):
        self.lib.ref_level_shape(self.handle, l, nx, ny)

    def lib_call(self, name, *args):
        st = getattr(self.lib, "ref_" + name)(self.handle, *args)
        if st:
            raise CheckerError(st, "reference call failed")
        return st

    def __del__(self):
        if getattr(self, "handle", None):
            self.lib.ref_problem_destroy(self.handle)
            self.handle = None

    def smooth_step(self, level, kind, smoother_omega, omega_damp, x, b):
        out = np.zeros(self.n(level))
        err = C.create_string_buffer(256)
        st = self.lib.ref_smooth_step(self.handle, level, SMOOTHERS.index(kind), smoother_omega,
                                      omega_damp, _ptr(np.ascontiguousarray(x, np.float64)),
                                      _ptr(np.ascontiguousarray(b, np.float64)), _ptr(out), err, 256)
        if st:
            raise CheckerError(st, err.value.decode())
        return out

    def adaptive_omega(self, level, d, corr):
        w = np.zeros(1)
        err = C.create_string_buffer(256)
        st = self.lib.ref_adaptive_omega(self.handle, level, _ptr(np.ascontiguousarray(d, np.float64)),
                                         _ptr(np.ascontiguousarray(corr, np.float64)), _ptr(w), err, 256)
        if st:
            raise CheckerError(st, err.value.decode())
        return float(w[0])

    def norm_l2(self, v, level=None):
        level = level or self.levels
        v = np.ascontiguousarray(v, np.float64)
        return self.lib.ref_norm_l2(self.handle, level, _ptr(v))

    def dot(self, a, b, level=None):
        level = level or self.levels
        return self.lib.ref_dot(self.handle, level, _ptr(np.ascontiguousarray(a, np.float64)),
                                _ptr(np.ascontiguousarray(b, np.float64)))

    def mg_cycle(self, spec: CycleSpec, level, u0, g):
        u = np.zeros(self.n(level))
        cs = spec.to_c()
        err = C.create_string_buffer(256)
        st = self.lib.ref_mg_cycle(self.handle, C.byref(cs), level,
                                   _ptr(np.ascontiguousarray(u0, np.float64)),
                                   _ptr(np.ascontiguousarray(g, np.float64)), _ptr(u), err, 256)
        if st:
            raise CheckerError(st, err.value.decode())
        return u

    def solve(self, spec: CycleSpec, b, x):
        hist = np.zeros(spec.max_cycles + 1)
        hl, it, cv = C.c_int(), C.c_int(), C.c_int()
        wall = np.zeros(1)
        err = C.create_string_buffer(256)
        cs = spec.to_c()
        st = self.lib.ref_solve(self.handle, C.byref(cs), _ptr(np.ascontiguousarray(b, np.float64)),
                                _ptr(x), _ptr(hist), C.byref(hl), C.byref(it), C.byref(cv),
                                _ptr(wall), err, 256)
        return SolveResult(st, hist[: hl.value].tolist(), it.value, bool(cv.value), float(wall[0]),
                           err.value.decode())

    def start_vector(self, spec: CycleSpec, kind, b):
        """gmg::make_start_vector (study.cpp:40-79); kind "zero" or "nested"."""
        x = np.zeros(self.n(self.levels))
        cs = spec.to_c()
        err = C.create_string_buffer(256)
        st = self.lib.ref_start_vector(self.handle, C.byref(cs), START_KINDS.index(kind),
                                       _ptr(np.ascontiguousarray(b, np.float64)), _ptr(x), err, 256)
        if st:
            raise CheckerError(st, err.value.decode())
        return x

    @classmethod
    def random_vector(cls, n, seed):
        v = np.zeros(n)
        cls.load().ref_random_vector(n, seed, _ptr(v))
        return v
