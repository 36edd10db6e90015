// Explicit instantiation lists of the heavy streaming-kernel templates, so the
// library builds as several translation units in parallel (build.py): solver.cu
// sees every list as `extern template` (the launch helpers only reference the
// host stubs), and each inst_*.cu defines GMG_INST_GROUP = one group and emits
// that group's device code. A combination missing here still works: solver.cu
// then instantiates it implicitly itself (slower build, same code).
#pragma once

#include "march.cuh"
#include "march2.cuh"
#include "march4.cuh"

namespace gmg_dev {

#define GMG_SM4(X, M, SK, C) \
    X __global__ void k_smooth4<M, SK, C>(Grid, C, const double*, Prolong, OmegaSrc, const double*, double*, double, int);
#define GMG_SM4_SK(X, M, C) GMG_SM4(X, M, 0, C) GMG_SM4(X, M, 1, C) GMG_SM4(X, M, 2, C) GMG_SM4(X, M, 3, C)
#define GMG_SM4_ALL(X, C) \
    GMG_SM4_SK(X, 0, C) GMG_SM4_SK(X, 1, C) GMG_SM4_SK(X, 2, C) GMG_SM4_SK(X, 3, C) GMG_SM4_SK(X, 4, C)

#define GMG_RES4(X, C)                                                                                        \
    X __global__ void k_resid4<false, C>(Grid, C, const double*, const double*, const double*, double*, double*, \
                                         Grid, RestrictW, double*, int);                                      \
    X __global__ void k_resid4<true, C>(Grid, C, const double*, const double*, const double*, double*, double*,  \
                                        Grid, RestrictW, double*, int);                                       \
    X __global__ void k_omega4<C>(Grid, C, Prolong, const double*, double*, double*, int*, int);

// group 1: CoefAxes smoothers; 2: CoefField smoothers; 3: the other smoothers;
// 4: residual / omega-term kernels of every class
#define GMG_GROUP1(X) GMG_SM4_ALL(X, CoefAxes)
#define GMG_GROUP2(X) GMG_SM4_ALL(X, CoefField)
#define GMG_GROUP3(X) GMG_SM4_ALL(X, CoefIso) GMG_SM4_ALL(X, CoefUnitSN) GMG_SM4_ALL(X, CoefConst) GMG_SM4_ALL(X, CoefRowX)
#define GMG_GROUP4(X)                                                                                     \
    GMG_RES4(X, CoefIso) GMG_RES4(X, CoefUnitSN) GMG_RES4(X, CoefConst) GMG_RES4(X, CoefRowX) GMG_RES4(X, CoefAxes) \
        GMG_RES4(X, CoefField)

#ifdef GMG_INST_GROUP
#define GMG_PASTE2(a, b) a##b
#define GMG_PASTE(a, b) GMG_PASTE2(a, b)
GMG_PASTE(GMG_GROUP, GMG_INST_GROUP)(template)
#else
GMG_GROUP1(extern template)
GMG_GROUP2(extern template)
GMG_GROUP3(extern template)
GMG_GROUP4(extern template)
#endif

}  // namespace gmg_dev
