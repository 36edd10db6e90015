"""B200-native geometric-multigrid F-cycle (drop-in for the gmg2d reference's solve path).

The compute path is libgmg_b200.so (hand-written sm_100a CUDA kernels behind the
C ABI in include/gmg_b200.h); paper_0805_3041_b200.gmg mirrors the reference's
C++ API in Python over that ABI.
"""
from .gmg import (CycleSpec, DivergenceError, GmgRuntimeError, InvalidArgument, LogicError,  # noqa: F401
                  MultilevelProblem, SolveReport, Unsupported, adaptive_omega, apply, axpy,
                  coarse_solve, dot, mg_cycle, norm_l2, prolongation, random_vector, residual,
                  restriction, smooth_step, solve, solve_device)
