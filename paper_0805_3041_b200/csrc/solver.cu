// B200-native geometric multigrid: device problem, cycle driver, C ABI.
//
// The cycle driver mirrors gmg::solve / fcycle_pass / mg_cycle
// (/root/reference/proj/src/cycle.cpp:69-194) but is executed as a CUDA graph:
// one F-cycle (defect cascade, coarse solve, one V-cycle per level with the
// adaptive correction weight computed on the device, the x+e update, the new
// residual and its exact-order norm) is captured once per cycle spec and
// replayed; the host only reads back the residual norm to run the reference's
// stopping and divergence tests.
#include <cuda_runtime.h>
#include <dlfcn.h>

#include <algorithm>
#include <array>
#include <chrono>
#include <climits>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <map>
#include <memory>
#include <mutex>
#include <random>
#include <set>
#include <stdexcept>
#include <string>
#include <thread>
#include <vector>

#include "../../include/gmg_b200.h"
#include "common.cuh"
#include "host_setup.h"
#include "dalloc.h"
#include "gs.cuh"
#include "linesm.cuh"
#include "march.cuh"
#include "march2.cuh"
#include "march4.cuh"
#include "inst.h"
#include "seqsum.cuh"
#include "vsmall.cuh"

using namespace gmg_dev;

namespace {

thread_local std::string g_last_error;

struct GmgError {
    int code;
    std::string msg;
};

#define CK(x)                                                                                  \
    do {                                                                                       \
        cudaError_t e_ = (x);                                                                  \
        if (e_ != cudaSuccess)                                                                 \
            throw GmgError{GMG_ERR_CUDA, std::string(#x) + " (solver.cu:" + std::to_string(__LINE__) + \
                                             "): " + cudaGetErrorString(e_)};                 \
    } while (0)

// after a launch: the launch error, and with GMG_DEBUG_SYNC the kernel's own
// completion status (debugging: pinpoints a faulting launch by line)
static const bool g_debug_sync = getenv("GMG_DEBUG_SYNC") != nullptr;
// GMG_NO_STAGE=1: pageable host vectors go through the runtime's own pageable copy (A/B knob)
static const bool g_no_stage = getenv("GMG_NO_STAGE") != nullptr;
// staged transfers of pageable host vectors (staged_rows)
constexpr int kStageThreads = 8, kStageSlots = 2;
// host threads that copy: GMG_STAGE_THREADS, default half the host's cores up to 8
// (C4 round trip of 1.6 GB on a 16-core box: 2/4/6/8 threads = 92/64/51/46 ms; pinned buffers 29 ms)
static const int g_stage_threads = [] {
    const char* e = getenv("GMG_STAGE_THREADS");
    const int n = e ? atoi(e) : (int)std::thread::hardware_concurrency() / 2;
    return std::max(1, std::min(kStageThreads, n));
}();
constexpr size_t kStageBytes = 4u << 20;  // per slot
constexpr size_t kStageMin = 32u << 20;   // smaller vectors take the plain copy
inline void dbg_sync(int line) {
    const cudaError_t e = cudaDeviceSynchronize();
    if (e != cudaSuccess)
        throw GmgError{GMG_ERR_CUDA, "debug sync after solver.cu:" + std::to_string(line) + ": " + cudaGetErrorString(e)};
}
#define KCHECK()                                        \
    do {                                                \
        CK(cudaGetLastError());                         \
        if (g_debug_sync) dbg_sync(__LINE__);           \
    } while (0)

// Every kernel is launched with the programmatic-dependent-launch attribute (the
// kernels start with pdl_wait()/pdl_trigger(), common.cuh): captured into the
// cycle graph as programmatic edges, so each launch overlaps its predecessor's
// tail. GMG_NO_PDL=1 launches plainly (A/B).
static const bool g_pdl = getenv("GMG_NO_PDL") == nullptr;

// Per-launch profile of one cycle run outside the graph (gmg_dev_profile_cycle):
// the launch helpers tag each launch with its kernel, level and algorithmic
// bytes (SURVEY.md §8d per-kernel bytes x the DOFs it covers); launch_k brackets
// it with events on the launching stream.
struct ProfEntry {
    std::string kernel;
    int level;
    double bytes;
    cudaEvent_t e0, e1;
};
thread_local std::vector<ProfEntry>* g_prof = nullptr;
thread_local std::string g_prof_kernel;
thread_local int g_prof_level = 0;
thread_local double g_prof_bytes = 0.0;
thread_local int g_cur_level = 0;  // level of the sums the driver is about to launch
inline void prof_tag(const char* kernel, int level, double bytes) {
    if (!g_prof) return;
    g_prof_kernel = kernel;
    g_prof_level = level;
    g_prof_bytes = bytes;
}

template <typename... KArgs, typename... Args>
void launch_k(void (*k)(KArgs...), dim3 grid, dim3 block, size_t smem, cudaStream_t st, Args&&... args) {
    if (g_prof) {
        ProfEntry e{g_prof_kernel.empty() ? std::string("other") : g_prof_kernel, g_prof_level, g_prof_bytes,
                    nullptr, nullptr};
        g_prof_kernel.clear();
        g_prof_bytes = 0.0;
        CK(cudaEventCreate(&e.e0));
        CK(cudaEventCreate(&e.e1));
        CK(cudaEventRecord(e.e0, st));
        g_prof->push_back(e);
    }
    cudaLaunchConfig_t cfg{};
    cfg.gridDim = grid;
    cfg.blockDim = block;
    cfg.dynamicSmemBytes = smem;
    cfg.stream = st;
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    at[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = at;
    cfg.numAttrs = g_pdl ? 1 : 0;
    CK(cudaLaunchKernelEx(&cfg, k, static_cast<KArgs>(std::forward<Args>(args))...));
    if (g_prof) CK(cudaEventRecord(g_prof->back().e1, st));
}

template <class F>
int guarded(F&& f) {
    try {
        f();
        return GMG_OK;
    } catch (const GmgError& e) {
        g_last_error = e.msg;
        return e.code;
    } catch (const std::invalid_argument& e) {
        g_last_error = e.what();
        return GMG_ERR_INVALID;
    } catch (const std::logic_error& e) {
        g_last_error = e.what();
        return GMG_ERR_LOGIC;
    } catch (const std::bad_alloc&) {
        g_last_error = "host allocation failed";
        return GMG_ERR_CUDA;
    } catch (const std::runtime_error& e) {
        g_last_error = e.what();
        return GMG_ERR_RUNTIME;
    }
}

enum Buf { U0 = 0, U1 = 1, DCAS = 2, GRHS = 3, DD = 4, NBUF = 5 };

struct Lev {
    int l = 1, nx = 0, ny = 0;
    long long pitch = 0;
    size_t elems = 0, off0 = 0;
    double* mem = nullptr;
    double* buf[NBUF] = {};
    int kind = 2;
    CoefConst cconst{};
    CoefRowX crow{};
    CoefField cfield{};
    CoefAxes caxes{};
    gmg_host::AxisTables axt;  // host copy of the AXES tables (kind 3)
    double* coefmem = nullptr;
    double *tx = nullptr, *ty = nullptr;  // prolongation weights (this level as fine)
    RestrictW rw{};                       // restriction weights (this level as coarse)
    double* wmem = nullptr;
    std::vector<double> hx, hy;
    double* scr[2] = {nullptr, nullptr};  // smoother scratch (adi/gsadi/ilu0), allocated on demand
    double* scrmem = nullptr;
    int w0 = 0, w1 = 0;  // owned rows; [0, ny) unless the level is sharded
    int per = 0;         // periodic in y (polar theta): rows wrap (common.cuh Grid)
    // the warp-strip kernels (march4.cuh) march non-periodic rows only
    bool strips() const;
    Grid grid() const { return Grid{nx, ny, pitch, w0, w1, per}; }
    int rows() const { return w1 - w0; }
    long long n() const { return (long long)nx * ny; }
};

// Per-level device state of one SmootherSpec (gmg::setup, smoother.cpp:230-273).
struct SmLev {
    double* mem = nullptr;
    LineFactors fx{}, fy{};                                    // factor_lines_x / _y
    const double *lw = nullptr, *ls = nullptr, *dp = nullptr;  // factor_ilu0
    double rich = 0.0;                                         // richardson_omega()
};
struct SmSetup {
    int kind = 0;
    double omega = 0.0;
    std::vector<SmLev> lev;
};

// ---- NCCL, loaded on first use (only the row-slab multi-process mode needs it) ----
typedef struct {
    char internal[128];
} NcclId;
enum { kNcclFloat64 = 8 };
struct NcclApi {
    int (*getUniqueId)(NcclId*) = nullptr;
    int (*commInitRank)(void**, int, NcclId, int) = nullptr;
    int (*commDestroy)(void*) = nullptr;
    int (*send)(const void*, size_t, int, int, void*, cudaStream_t) = nullptr;
    int (*recv)(void*, size_t, int, int, void*, cudaStream_t) = nullptr;
    int (*bcast)(const void*, void*, size_t, int, int, void*, cudaStream_t) = nullptr;
    int (*allGather)(const void*, void*, size_t, int, void*, cudaStream_t) = nullptr;
    int (*groupStart)() = nullptr;
    int (*groupEnd)() = nullptr;
    const char* (*errStr)(int) = nullptr;
};

// Row-slab distribution shared by the slabs of one solve.
struct DistCtx {
    int world = 1;
    int Ls = 0;       // first sharded level
    int H = 4;        // halo rows exchanged (>= fused smoothing steps per launch)
    bool local = true;  // virtual ranks: all slabs in this process on one stream
    void* comm = nullptr;  // ncclComm_t (multi-process mode)
    std::vector<gmg_problem*> slabs;  // local mode: slab r = rank r (slab 0 owns the others)
    std::vector<std::vector<int>> w0, w1;  // [level-1][rank]
    ~DistCtx();
};

}  // namespace

struct gmg_problem {
    int L = 0, device = 0;
    cudaStream_t st = nullptr;
    std::mutex mu;
    std::vector<Lev> lv;
    double* xmem = nullptr;
    double* X[2] = {nullptr, nullptr};
    double* B = nullptr;
    double* band = nullptr;
    double* cscr = nullptr;
    int cn = 0, cbw = 0;
    // exact-order summation workspace
    int nch_max = 0;
    double* csum = nullptr;          // fast-mode partials [2][nch]
    double* T = nullptr;             // materialised omega terms, 2 x N_L dense
    double* lb = nullptr;            // look-back values: per sum agg, incl [nch] each
    unsigned char* lbs = nullptr;    // per sum: cagg, cincl [nch] ChunkAgg each
    int* flags = nullptr;            // per sum: ticket, total, flag[nch], cflag[nch]
    gmg_ss::Rec* recs = nullptr;     // per sum: rec_cap records (per-chunk slots)
    gmg_ss::Rec* recs2 = nullptr;    // per sum: rec_cap records (compacted, in order)
    int rec_cap = 0;
    bool ss_clean = false;  // exact-sum flags known zero (the last walk ended in a fused scan+chain)
    // "correction nonzero" flags of adaptive omega, one slot per level visit of a cycle
    // (reset by one memset per cycle instead of one per visit); nz_cur: the current visit's
    static constexpr int kNzSlots = 1024;
    int* nz_slots = nullptr;
    int nz_next = 0;
    int* nz_cur = nullptr;
    unsigned long long* ss_stats = nullptr;  // [16] exact-sum engine counters (seqsum.cuh)
    longlong2* gs_edge = nullptr;            // Gauss-Seidel wavefront warp-edge rows: {value, generation} words
    long long* gs_state = nullptr;           // {generation, finished-CTA count} (gs.cuh)
    int gs_epitch = 0;
    int gs_warps = 0;
    double* sums = nullptr;  // [0..1] omega sums, [2] residual norm^2, [3] misc
    int* nz = nullptr;
    int* status = nullptr;
    double* hostbuf = nullptr;  // pinned: {norm^2, status}
    char* stage = nullptr;      // pinned ring for pageable host vectors (staged_rows), allocated on first use
    bool stage_failed = false;  // the host refused to pin the ring: plain pageable copies
    cudaEvent_t stage_ev[kStageThreads * kStageSlots] = {};
    std::map<std::string, std::array<cudaGraphExec_t, 2>> graphs;
    std::map<std::pair<int, unsigned long long>, SmSetup> smsetups;  // (kind, omega bits)
    double* linebuf = nullptr;  // k_gstri scratch: 2 x max(nx, ny)
    // row-slab mode: rank of this slab and the shared context (null: single GPU)
    int rank = 0;
    bool owns_stream = true;
    std::shared_ptr<DistCtx> dist;
    double* dscr = nullptr;  // [0,8): approx totals + nz; [8,16): rank prefix; [16,24): start; [32,..): gathered
    cudaEvent_t ev0 = nullptr, ev1 = nullptr;
    Lev& lev(int l) { return lv.at(l - 1); }
};

namespace {

// ---------------------------------------------------------------------------
// simple (non-streaming) kernels
// ---------------------------------------------------------------------------
__global__ void k_restrict_simple(Grid fg, const double* __restrict__ f, Grid cg, RestrictW rw,
                                  double* __restrict__ c) {
    pdl_wait();  // programmatic dependent launch: inputs of the previous kernel are complete
    pdl_trigger();
    const int P = blockIdx.x * blockDim.x + threadIdx.x;
    const int Q = blockIdx.y * blockDim.y + threadIdx.y;
    if (P >= cg.nx || Q >= cg.ny) return;
    c[cg.at(P, Q)] = restrict_at(rw, P, Q, [&](int di, int dj) {
        return __ldg(f + fg.at(2 * P + 1 + di, 2 * Q + 1 + dj));
    });
}

__global__ void k_prolong_simple(Prolong P, Grid fg, double* __restrict__ out) {
    pdl_wait();  // programmatic dependent launch: inputs of the previous kernel are complete
    pdl_trigger();
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    const int j = blockIdx.y * blockDim.y + threadIdx.y;
    if (i >= fg.nx || j >= fg.ny) return;
    out[fg.at(i, j)] = P.at(i, j);
}

template <class Coef>
__global__ void k_apply_simple(Grid g, Coef A, const double* __restrict__ x, double* __restrict__ y) {
    pdl_wait();  // programmatic dependent launch: inputs of the previous kernel are complete
    pdl_trigger();
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    const int j = blockIdx.y * blockDim.y + threadIdx.y;
    if (i >= g.nx || j >= g.ny) return;
    auto X = [&](int a, int b) { return g.inside(a, b) ? __ldg(x + g.at(a, b)) : 0.0; };
    y[g.at(i, j)] = stencil_apply(A, i, j, X(i, j), X(i - 1, j), X(i + 1, j), X(i, j - 1), X(i, j + 1));
}

__global__ void k_axpy_flat(long long n, double a, const double* __restrict__ x, double* __restrict__ y) {
    pdl_wait();  // programmatic dependent launch: inputs of the previous kernel are complete
    pdl_trigger();
    const long long k = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    if (k < n) y[k] = y[k] + a * x[k];
}

// BandedCholesky::solve (stencil.cpp:190-210): forward then backward
// substitution in the reference's d-loop order, one thread (level 1 is tiny).
__global__ void k_coarse_chol(const double* __restrict__ band, int n, int bw, Grid g,
                              const double* __restrict__ b, double* __restrict__ x,
                              double* __restrict__ xs) {
    pdl_wait();  // programmatic dependent launch: inputs of the previous kernel are complete
    pdl_trigger();
    if (threadIdx.x != 0 || blockIdx.x != 0) return;
    for (int k = 0; k < n; ++k) {
        double acc = b[g.at(k % g.nx, k / g.nx)];
        const int dm = min(bw, k);
        for (int d = 1; d <= dm; ++d) acc = acc - band[(long long)d * n + k] * xs[k - d];
        xs[k] = acc / band[k];
    }
    for (int k = n - 1; k >= 0; --k) {
        double acc = xs[k];
        const int dm = min(bw, n - 1 - k);
        for (int d = 1; d <= dm; ++d) acc = acc - band[(long long)d * n + k + d] * xs[k + d];
        xs[k] = acc / band[k];
    }
    for (int k = 0; k < n; ++k) x[g.at(k % g.nx, k / g.nx)] = xs[k];
}

// Fast (tree-order) reduction finisher: sums the chunk partials of S1.
__global__ void k_fast_final(const double* __restrict__ csum, int nch, int ns, double* __restrict__ out,
                             const double* __restrict__ start) {
    pdl_wait();  // programmatic dependent launch: inputs of the previous kernel are complete
    pdl_trigger();
    __shared__ double red[32];
    for (int s = 0; s < ns; ++s) {
        double a = 0.0;
        for (int c = threadIdx.x; c < nch; c += blockDim.x) a += csum[(long long)s * nch + c];
        for (int o = 16; o > 0; o >>= 1) a += __shfl_xor_sync(0xffffffffu, a, o);
        if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = a;
        __syncthreads();
        if (threadIdx.x == 0) {
            double t = 0.0;
            for (int w = 0; w < (int)(blockDim.x >> 5); ++w) t += red[w];
            out[s] = start ? start[s] + t : t;
        }
        __syncthreads();
    }
}

// adaptive_omega on two explicit arrays (unit op): writes (A corr)_k corr_k and
// d_k corr_k densely, and whether some corr_k^2 != 0.
template <class Coef>
__global__ void k_omega_terms_field(Grid g, Coef A, const double* __restrict__ d, const double* __restrict__ cr,
                                    double* __restrict__ T0, double* __restrict__ T1, int* __restrict__ nz) {
    pdl_wait();  // programmatic dependent launch: inputs of the previous kernel are complete
    pdl_trigger();
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    const int j = blockIdx.y * blockDim.y + threadIdx.y;
    if (i >= g.nx || j >= g.ny) return;
    auto C = [&](int a, int b) { return g.inside(a, b) ? __ldg(cr + g.at(a, b)) : 0.0; };
    const double cc = C(i, j);
    const double ac = stencil_apply(A, i, j, cc, C(i - 1, j), C(i + 1, j), C(i, j - 1), C(i, j + 1));
    const long long k = (long long)j * g.nx + i;
    T0[k] = ac * cc;
    T1[k] = __ldg(d + g.at(i, j)) * cc;
    if ((cc * cc) != 0.0) atomicOr(nz, 1);
}

// ---------------------------------------------------------------------------
// launch helpers
// ---------------------------------------------------------------------------
constexpr int kTW = 128;

// Rows per CTA segment: halved from 128 until the grid has >= 32*148 warp strips
// (GMG_SEG_TARGET), i.e. about two full waves at 16 resident warps per SM; short segments so
// the grid has enough CTAs and each marches few rows (the march is latency-bound
// per row). Always even (the restriction pairs fine rows).
int seg_rows(int nx, int ny) {
    static const long long target = [] {
        const char* e = getenv("GMG_SEG_TARGET");
        return e ? atoll(e) : 32LL * 148;  // warps: ~2 full waves of the 16-warp/SM streaming kernels
    }();
    static const int seg_min_big = [] {
        const char* e = getenv("GMG_SEG_MIN");
        return e ? atoi(e) : 8;
    }();
    // GMG_SEG_FORCE="nx:seg,nx:seg": rows per segment for levels of that width (tuning sweeps)
    static const std::map<int, int> forced = [] {
        std::map<int, int> m;
        if (const char* e = getenv("GMG_SEG_FORCE")) {
            int a = 0, b = 0, nch = 0;
            while (sscanf(e, "%d:%d%n", &a, &b, &nch) == 2) {
                m[a] = std::max(2, b & ~1);
                e += nch;
                if (*e == ',') ++e;
            }
        }
        return m;
    }();
    if (auto it = forced.find(nx); it != forced.end()) return it->second;
    const int strips = (nx + 123) / 124;
    // large levels (the warp-strip kernels): segments no shorter than seg_min_big rows, so the
    // 2M-row vertical halo of a fused smoothing launch stays a small share of the march
    static const int seg_min_small = [] {
        const char* e = getenv("GMG_SEG_MIN_SMALL");
        return e ? atoi(e) : 2;  // small levels: short marches win (measured 8 -> 2: -1.3% per C4 cycle)
    }();
    const int smin = nx >= 255 ? seg_min_big : seg_min_small;
    int seg = 128;
    while (seg > smin && (long long)strips * ((ny + seg - 1) / seg) < target) seg /= 2;
    // One resident wave: if longer segments make the whole grid fit the SMs at once (4 CTAs of
    // 4 strips per SM) and nearly fill them, take them — no second-wave tail, and the 2M halo
    // rows and the start-up latency of a segment are paid less often (4095^2: 16 -> 64 rows,
    // -1.0% per C4 cycle, -0.3% per C5 cycle; no other level of the configs qualifies).
    if (nx >= 255) {
        static const long long resident = [] {
            int dev = 0, sms = 148;
            cudaGetDevice(&dev);
            cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
            return 4LL * sms;
        }();
        const long long ctax = (strips + 3) / 4;
        for (int s2 = 128; s2 > seg; s2 /= 2) {
            const long long n = ctax * ((ny + s2 - 1) / s2);
            if (n <= resident && 10 * n >= 8 * resident) return s2;
        }
    }
    return seg;
}

template <class F>
void with_coef(const Lev& L, F&& f) {
    if (L.kind == 0) f(L.cconst);
    else if (L.kind == 1) f(L.crow);
    else if (L.kind == 3) f(L.caxes);
    else f(L.cfield);
}

// Coefficient classes of the warp-strip kernels (large levels): constant rows
// specialised when their legs are exactly -1 (common.cuh CoefIso / CoefUnitSN).
template <class F>
void with_coef_big(const Lev& L, F&& f) {
    if (L.kind == 0) {
        const CoefConst& k = L.cconst;
        if (k.c_pow2 && k.w == -1.0 && k.e == -1.0 && k.s == -1.0 && k.n == -1.0) {
            CoefIso A;
            static_cast<CoefConst&>(A) = k;
            f(A);
            return;
        }
        if (k.s == -1.0 && k.n == -1.0 && k.rcp_ok) {
            CoefUnitSN A;
            static_cast<CoefConst&>(A) = k;
            f(A);
            return;
        }
    }
    with_coef(L, f);
}

// Once-per-device setup (function attributes apply to the current device only):
// a (key, device) set guarded by a mutex, so problems on several devices and
// concurrent creates/solves on different threads each configure their device.
bool first_on_device(const void* key) {
    static std::mutex mu;
    static std::set<std::pair<const void*, int>> done;
    int dev = 0;
    CK(cudaGetDevice(&dev));
    std::lock_guard<std::mutex> lk(mu);
    return done.insert({key, dev}).second;
}

// Dynamic shared memory opt-in of kernel fn on the current device (once per device).
template <class T>
void set_smem(T* fn, size_t bytes) {
    if (!first_on_device(reinterpret_cast<const void*>(fn))) return;
    CK(cudaFuncSetAttribute(reinterpret_cast<const void*>(fn), cudaFuncAttributeMaxDynamicSharedMemorySize,
                            (int)bytes));
}

// sums up to this length walk in small chunks (GMG_SS_SMALL_MAX overrides, for A/B timing)
long long ss_small_max() {
    static const long long v = [] {
        const char* e = getenv("GMG_SS_SMALL_MAX");
        return e ? atoll(e) : kSsSmallMax;
    }();
    return v;
}

SsPair ss_state(gmg_problem* p, int nch) {
    SsPair sp{};
    for (int s = 0; s < kSsMaxSums; ++s) {
        SsState& S = sp.s[s];
        int* f = p->flags + (size_t)s * (2 + 2 * (size_t)p->nch_max);
        S.ticket = f;
        S.total = f + 1;
        S.flag = f + 2;
        S.cflag = f + 2 + nch;
        S.lbw = reinterpret_cast<longlong2*>(p->lb + (size_t)s * 2 * p->nch_max);
        S.cagg = p->lbs + (size_t)s * 2 * p->nch_max * sizeof(ChunkAgg);
        S.cincl = S.cagg + (size_t)p->nch_max * sizeof(ChunkAgg);
        S.recs = p->recs + (size_t)s * p->rec_cap;
        S.recs2 = p->recs2 + (size_t)s * p->rec_cap;
        S.stats = p->ss_stats;

    }
    return sp;
}

template <class TG>
void seqsum_attrs() {
    set_smem(k_ss_walk<TG, kSsEPT>, ss_walk_smem<kSsEPT>());
    set_smem(k_ss_walk<TG, kSsEPTs>, ss_walk_smem<kSsEPTs>());
    set_smem(k_ss_chain<TG>, ss_chain_smem());
    set_smem(k_ss_scan_chain<TG>, ss_chain_smem());
}

// Loads (lazy module loading) and configures every exact-sum kernel before any
// graph capture, so no kernel is first touched while a stream is capturing.
void preload_seqsum_kernels() {
    static const char key = 0;
    if (!first_on_device(&key)) return;
    seqsum_attrs<NormTerms>();
    seqsum_attrs<ArrTerms>();
    seqsum_attrs<DotTerms>();
    seqsum_attrs<FlatNormTerms>();
    cudaFuncAttributes fa;
    CK(cudaFuncGetAttributes(&fa, k_ss_scan2));
    CK(cudaFuncGetAttributes(&fa, k_ss_direct<NormTerms>));
    CK(cudaFuncGetAttributes(&fa, k_ss_direct<ArrTerms>));
    CK(cudaFuncGetAttributes(&fa, k_ss_direct<DotTerms>));
    CK(cudaFuncGetAttributes(&fa, k_ss_direct<FlatNormTerms>));
}

// Sums of TG's NS term sequences, each bit-identical to the reference's
// left-to-right loop (mode EXACT) or in tree order (mode FAST); out[s].
// start (device, NS values, may be null): exact state entering the range, i.e.
// the sum of the terms before it (earlier row slabs); pre0: an approximation of
// the same, used only to seed the speculative walk. Split in two phases so
// that row slabs can run their walks concurrently and chain in rank order.
// fused_out != null: the chain runs inside the scan kernel (k_ss_scan_chain) and writes the
// NS sums there, starting from fused_start (may be null).
template <class TG>
void seqsum_walk(gmg_problem* p, const TG& tg, long long n, const double* pre0, double* fused_out = nullptr,
                 const double* fused_start = nullptr) {
    constexpr int NS = TG::NS;
    const bool small = n <= ss_small_max();
    const int cs = small ? kSsCs : kSsC;
    const int nch = (int)((n + cs - 1) / cs);
    if (nch > p->nch_max) throw GmgError{GMG_ERR_LOGIC, "seqsum: workspace too small"};
    seqsum_attrs<TG>();
    if (n <= kSsDirect) return;  // the direct kernel needs no walk
    const SsPair sp = ss_state(p, nch);
    // A fused scan+chain leaves the flags it used zeroed; after the split path (row
    // slabs) they are dirty and the whole per-sum flag region is cleared (a later sum
    // with more chunks reads further into it).
    if (!(fused_out && p->ss_clean))
        for (int s = 0; s < NS; ++s)
            CK(cudaMemsetAsync(sp.s[s].ticket, 0, (2 + 2 * (size_t)p->nch_max) * sizeof(int), p->st));
    p->ss_clean = fused_out != nullptr;
    prof_tag(TG::kProfName, g_cur_level, (double)n * TG::kBytesPerTerm);
    if (small)
        launch_k(k_ss_walk<TG, kSsEPTs>, dim3(nch, NS), kSsWT, ss_walk_smem<kSsEPTs>(), p->st, tg, n, nch, sp, pre0);
    else
        launch_k(k_ss_walk<TG, kSsEPT>, dim3(nch, NS), kSsWT, ss_walk_smem<kSsEPT>(), p->st, tg, n, nch, sp, pre0);
    const dim3 sg((nch + kSsScanB - 1) / kSsScanB, NS);
    prof_tag(fused_out ? "ss_scan_chain" : "ss_scan", g_cur_level, 0.0);
    if (fused_out)
        launch_k(k_ss_scan_chain<TG>, sg, kSsScanB, ss_chain_smem(), p->st, tg, n, sp, nch, fused_out, fused_start);
    else
        launch_k(k_ss_scan2, sg, kSsScanB, 0, p->st, sp, nch);
    KCHECK();
}

template <class TG>
void seqsum_chain(gmg_problem* p, const TG& tg, long long n, double* out, const double* start) {
    constexpr int NS = TG::NS;
    if (n == 0) {  // the reference's loop leaves s unchanged (0.0 for a whole sum)
        if (start)
            CK(cudaMemcpyAsync(out, start, NS * sizeof(double), cudaMemcpyDeviceToDevice, p->st));
        else
            CK(cudaMemsetAsync(out, 0, NS * sizeof(double), p->st));
            if (g_debug_sync) dbg_sync(__LINE__);
        return;
    }
    if (n <= kSsDirect) {
        prof_tag("ss_direct", g_cur_level, (double)n * TG::kBytesPerTerm);
        launch_k(k_ss_direct<TG>, NS, 256, n * sizeof(double), p->st, tg, (int)n, out, start);
        KCHECK();
        return;
    }
    const int nch = (int)((n + kSsC - 1) / kSsC);
    const SsPair sp = ss_state(p, nch);
    prof_tag("ss_chain", g_cur_level, 0.0);
    launch_k(k_ss_chain<TG>, NS, kSsT, ss_chain_smem(), p->st, tg, n, sp, out, start);
    KCHECK();
}

// tree-order partial sums of the NS sequences into out (fast mode; also the
// approximate totals that seed the walks of later row slabs)
template <class TG>
void seqsum_fast(gmg_problem* p, const TG& tg, long long n, double* out, const double* start) {
    constexpr int NS = TG::NS;
    const int nch = (int)((n + kSsPC - 1) / kSsPC);  // partial-sum CTAs (kSsT threads x kSsEPT terms)
    if (nch > p->nch_max) throw GmgError{GMG_ERR_LOGIC, "seqsum: workspace too small"};
    if (n == 0) {
        if (start)
            CK(cudaMemcpyAsync(out, start, NS * sizeof(double), cudaMemcpyDeviceToDevice, p->st));
        else
            CK(cudaMemsetAsync(out, 0, NS * sizeof(double), p->st));
            if (g_debug_sync) dbg_sync(__LINE__);
        return;
    }
    launch_k(k_ss_partial<TG>, dim3(nch, NS), kSsT, 0, p->st, tg, n, p->csum, nch);
    launch_k(k_fast_final, 1, 1024, 0, p->st, p->csum, nch, NS, out, start);
    KCHECK();
}

template <class TG>
void seqsum(gmg_problem* p, const TG& tg, long long n, double* out, int mode, const double* start = nullptr,
            const double* pre0 = nullptr) {
    if (mode == GMG_REDUCE_FAST) {
        seqsum_fast(p, tg, n, out, start);
        return;
    }
    if (n <= kSsDirect) {  // the direct kernel (or the empty sum): no walk
        seqsum_chain(p, tg, n, out, start);
        return;
    }
    static const bool split = getenv("GMG_SPLIT_CHAIN") != nullptr;  // A/B: separate chain launch
    if (split) {
        seqsum_walk(p, tg, n, pre0);
        seqsum_chain(p, tg, n, out, start);
        return;
    }
    seqsum_walk(p, tg, n, pre0, out, start);
}

Prolong prolong_from(gmg_problem* p, int coarse_level, const double* uc) {
    const Lev& C = p->lev(coarse_level);
    const Lev& F = p->lev(coarse_level + 1);
    return Prolong{uc, C.grid(), F.tx, F.ty};
}

enum Start { S_ZERO = 0, S_U = 1, S_PROLONG = 2, S_CORRECT = 3, S_SUM = 4 };

struct SmoothSrc {
    Start kind = S_ZERO;
    const double* u = nullptr;   // S_U, S_CORRECT
    const double* uc = nullptr;  // S_PROLONG, S_CORRECT: coarse grid function (level l-1)
    OmegaSrc om{nullptr, nullptr, 1.0, nullptr};
};

template <int M, class Coef, class Src>
void launch_smooth2_t(gmg_problem* p, const Lev& L, const Coef& A, const Src& src, OmegaSrc om,
                      const double* g, double* out, double wd) {
    constexpr int H = (M + 1) & ~1;
    constexpr int OUTW = 2 * kTW - 2 * H;
    constexpr int PF = sizeof(typename Src::Raw) > 32 ? 2 : 3;
    const int seg = seg_rows(L.nx, L.rows());
    dim3 grid((L.nx + OUTW - 1) / OUTW, (L.rows() + seg - 1) / seg);
    prof_tag(Src::kProfName, L.l, Src::kBytesPerDof * (double)L.nx * L.rows());
    launch_k(k_smooth2<M, kTW, PF, Coef, Src>, grid, kTW, 0, p->st, L.grid(), A, src, om, g, out, wd, seg);
    KCHECK();
}

template <int M, int SK, class Coef>
void launch_smooth4_t(gmg_problem* p, const Lev& L, const Coef& A, const double* u, const double* uc,
                      OmegaSrc om, const double* g, double* out, double wd) {
    constexpr int H = (M + 1) & ~1;
    constexpr int OW = 128 - 2 * H;
    constexpr size_t smem = smooth4_smem<SK, M>();
    set_smem(k_smooth4<M, SK, Coef>, smem);
    Prolong P{};
    if (SK == K3_PROLONG || SK == K3_CORRECT) P = prolong_from(p, L.l - 1, uc);
    const int seg = seg_rows(L.nx, L.rows());
    const int strips = (L.nx + OW - 1) / OW;
    dim3 grid((strips + kS4W - 1) / kS4W, (L.rows() + seg - 1) / seg);
    {
        static const char* names[4] = {"smooth(from 0)", "smooth(from u)", "smooth(from P e)", "smooth(u + w P uc)"};
        static const double bpd[4] = {16.0, 24.0, 18.0, 26.0};  // §8d: g in + out (+u) (+ coarse N/4)
        prof_tag(names[SK], L.l, bpd[SK] * (double)L.nx * L.rows());
    }
    launch_k(k_smooth4<M, SK, Coef>, grid, kS4W * 32, smem, p->st, L.grid(), A, u, P, om, g, out, wd, seg);
    KCHECK();
}

// levels at least this wide use the warp-strip kernels (march4.cuh); GMG_RING_MIN_NX for A/B
static const int kRingMinNx = [] {
    const char* e = getenv("GMG_RING_MIN_NX");
    return e ? atoi(e) : 255;
}();
bool Lev::strips() const { return nx >= kRingMinNx && !per; }
template <int M, class Coef>
void launch_smooth_src(gmg_problem* p, const Lev& L, const Coef& A, const SmoothSrc& s, const double* g,
                       double* out, double wd) {
    if constexpr (std::is_same<Coef, CoefIso>::value || std::is_same<Coef, CoefUnitSN>::value) {
        switch (s.kind) {
            case S_ZERO: launch_smooth4_t<M, K3_ZERO>(p, L, A, nullptr, nullptr, s.om, g, out, wd); return;
            case S_U: launch_smooth4_t<M, K3_U>(p, L, A, s.u, nullptr, s.om, g, out, wd); return;
            case S_PROLONG: launch_smooth4_t<M, K3_PROLONG>(p, L, A, nullptr, s.uc, s.om, g, out, wd); return;
            case S_CORRECT: launch_smooth4_t<M, K3_CORRECT>(p, L, A, s.u, s.uc, s.om, g, out, wd); return;
            default: throw GmgError{GMG_ERR_LOGIC, "smooth: bad source"};
        }
    } else {
    if (L.strips()) {
        switch (s.kind) {
            case S_ZERO: launch_smooth4_t<M, K3_ZERO>(p, L, A, nullptr, nullptr, s.om, g, out, wd); return;
            case S_U: launch_smooth4_t<M, K3_U>(p, L, A, s.u, nullptr, s.om, g, out, wd); return;
            case S_PROLONG: launch_smooth4_t<M, K3_PROLONG>(p, L, A, nullptr, s.uc, s.om, g, out, wd); return;
            case S_CORRECT: launch_smooth4_t<M, K3_CORRECT>(p, L, A, s.u, s.uc, s.om, g, out, wd); return;
            default: throw GmgError{GMG_ERR_LOGIC, "smooth: bad source"};
        }
    }
    switch (s.kind) {
        case S_ZERO:
            launch_smooth2_t<M>(p, L, A, Src2Zero{}, s.om, g, out, wd);
            break;
        case S_U:
            launch_smooth2_t<M>(p, L, A, Src2U{s.u, L.grid()}, s.om, g, out, wd);
            break;
        case S_PROLONG: {
            Src2Prolong src{prolong_from(p, L.l - 1, s.uc), L.nx, L.ny, 0.0};
            launch_smooth2_t<M>(p, L, A, src, s.om, g, out, wd);
            break;
        }
        case S_CORRECT: {
            Src2Correct src{s.u, L.grid(), prolong_from(p, L.l - 1, s.uc), 0.0, 0.0};
            launch_smooth2_t<M>(p, L, A, src, s.om, g, out, wd);
            break;
        }
        default:
            throw GmgError{GMG_ERR_LOGIC, "smooth: bad source"};
    }
    }
}

// One launch of M <= 4 Jacobi steps.
void launch_smooth(gmg_problem* p, const Lev& L, int M, const SmoothSrc& s, const double* g, double* out,
                   double wd) {
    auto go = [&](const auto& A) {
        switch (M) {
            case 0: launch_smooth_src<0>(p, L, A, s, g, out, wd); break;
            case 1: launch_smooth_src<1>(p, L, A, s, g, out, wd); break;
            case 2: launch_smooth_src<2>(p, L, A, s, g, out, wd); break;
            case 3: launch_smooth_src<3>(p, L, A, s, g, out, wd); break;
            case 4: launch_smooth_src<4>(p, L, A, s, g, out, wd); break;
            default: throw GmgError{GMG_ERR_LOGIC, "smooth: M > 4"};
        }
    };
    if (L.strips()) with_coef_big(L, go);  // k_smooth4
    else with_coef(L, go);
}

constexpr int kMaxFuse = 4;

template <class Coef, class Src>
void launch_resid_t(gmg_problem* p, const Lev& L, const Coef& A, const Src& src, const double* g,
                    double* dout, double* x0out, double* gc, int neg = 0,
                    OmegaSrc om = OmegaSrc{nullptr, nullptr, 1.0, nullptr}) {
    const int seg = seg_rows(L.nx, L.rows());
    dim3 grid((L.nx + (kTW - 4) - 1) / (kTW - 4), (L.rows() + seg - 1) / seg);
    Grid cg{0, 0, 0};
    RestrictW rw{};
    if (gc) {
        const Lev& C = p->lev(L.l - 1);
        cg = C.grid();
        rw = C.rw;
    }
    constexpr int PF = sizeof(typename Src::Raw) > 16 ? 2 : 4;
    prof_tag(gc ? "residual+restrict" : "residual", L.l,
             (8.0 * (Src::kReads + 1) + 8.0 * ((dout != nullptr) + (x0out != nullptr)) + (gc ? 2.0 : 0.0)) *
                 (double)L.nx * L.rows());
    launch_k(k_resid<kTW, PF, Coef, Src>, grid, kTW, 0, p->st, L.grid(), A, src, g, dout, x0out, cg, rw, gc, seg, neg,
                                                          om);
    KCHECK();
}

template <bool SUM, class Coef>
void launch_resid4_t(gmg_problem* p, const Lev& L, const Coef& A, const double* u, const double* e, const double* g,
                     double* dout, double* x0out, double* gc) {
    constexpr size_t smem = resid4_smem<SUM>();
    set_smem(k_resid4<SUM, Coef>, smem);
    Grid cg{0, 0, 0};
    RestrictW rw{};
    if (gc) {
        const Lev& C = p->lev(L.l - 1);
        cg = C.grid();
        rw = C.rw;
    }
    const int seg = seg_rows(L.nx, L.rows());
    const int strips = (L.nx + 123) / 124;
    dim3 grid((strips + kS4W - 1) / kS4W, (L.rows() + seg - 1) / seg);
    prof_tag(SUM ? (gc ? "x+e, residual+restrict" : "x+e, residual") : (gc ? "residual+restrict" : "residual"), L.l,
             (8.0 * (SUM ? 3 : 2) + 8.0 * ((dout != nullptr) + (x0out != nullptr)) + (gc ? 2.0 : 0.0)) *
                 (double)L.nx * L.rows());
    launch_k(k_resid4<SUM, Coef>, grid, kS4W * 32, smem, p->st, L.grid(), A, u, e, g, dout, x0out, cg, rw, gc, seg);
    KCHECK();
}

// residual of (u, or x+e when e != null) against g; optional outputs.
void launch_resid(gmg_problem* p, const Lev& L, const double* u, const double* e, const double* g,
                  double* dout, double* x0out, double* gc) {
    if (L.strips()) {
        with_coef_big(L, [&](const auto& A) {
            if (e)
                launch_resid4_t<true>(p, L, A, u, e, g, dout, x0out, gc);
            else
                launch_resid4_t<false>(p, L, A, u, nullptr, g, dout, x0out, gc);
        });
        return;
    }
    with_coef(L, [&](const auto& A) {
        if (e)
            launch_resid_t(p, L, A, SrcSum{u, e, L.grid()}, g, dout, x0out, gc);
        else
            launch_resid_t(p, L, A, SrcU{u, L.grid()}, g, dout, x0out, gc);
    });
}

// Defect A x0 - g of a smoothing start (any source), optionally storing x0.
void launch_defect_src(gmg_problem* p, const Lev& L, const SmoothSrc& s, const double* g, double* dout,
                       double* x0out) {
    with_coef(L, [&](const auto& A) {
        switch (s.kind) {
            case S_ZERO:
                launch_resid_t(p, L, A, SrcZero{}, g, dout, x0out, nullptr, 1);
                break;
            case S_U:
                launch_resid_t(p, L, A, SrcU{s.u, L.grid()}, g, dout, x0out, nullptr, 1);
                break;
            case S_PROLONG:
                launch_resid_t(p, L, A, SrcProlong{prolong_from(p, L.l - 1, s.uc), L.nx, L.ny, 0.0}, g, dout,
                               x0out, nullptr, 1);
                break;
            case S_CORRECT:
                launch_resid_t(p, L, A, SrcCorrect{s.u, L.grid(), prolong_from(p, L.l - 1, s.uc), 0.0, 0.0}, g,
                               dout, x0out, nullptr, 1, s.om);
                break;
            default:
                throw GmgError{GMG_ERR_LOGIC, "defect: bad source"};
        }
    });
}

// One wavefront pass of policy `pol` (gs.cuh) over level L.
template <class Pol>
void launch_wave(gmg_problem* p, const Lev& L, const Pol& pol, const double* d, const double* x, double* xo,
                 double damp) {
    const int warps = (L.ny + 31) / 32;
    if (warps > p->gs_warps) throw GmgError{GMG_ERR_LOGIC, "gs: workspace too small"};
    const int blocks = (warps + kGsWarps - 1) / kGsWarps;
    if (blocks > 148) throw GmgError{GMG_ERR_UNSUPPORTED, "gs: more rows than one co-resident wavefront"};
    set_smem(k_gs_wave<Pol>, gs_smem());
    prof_tag("gs wavefront", L.l, (Pol::UPDATE ? 24.0 : 16.0) * (double)L.nx * L.ny);
    launch_k(k_gs_wave<Pol>, blocks, kGsThreads, gs_smem(), p->st, L.grid(), pol, d, x, xo, damp, p->gs_edge,
             p->gs_epitch, p->gs_state);
    KCHECK();
}

// One lexicographic Gauss-Seidel/SOR smooth_step: x' = x - damp * (D + om L)^{-1} (A x - g).
void launch_gs_wave(gmg_problem* p, const Lev& L, const double* d, const double* x, double* xo, double om,
                    double damp) {
    if (L.kind == 0) {  // constant operator: the division form is chosen here, not per point
        const CoefConst& A = L.cconst;
        if (A.c_pow2) launch_wave(p, L, GsPolicy<CoefConst, 1>{A, om}, d, x, xo, damp);
        else if (A.rcp_ok) launch_wave(p, L, GsPolicy<CoefConst, 2>{A, om}, d, x, xo, damp);
        else launch_wave(p, L, GsPolicy<CoefConst, 0>{A, om}, d, x, xo, damp);
        return;
    }
    with_coef(L, [&](const auto& A) {
        using C = std::decay_t<decltype(A)>;
        launch_wave(p, L, GsPolicy<C>{A, om}, d, x, xo, damp);
    });
}

bool uses_x_lines(int k) {
    return k == GMG_SMOOTHER_TRI_X || k == GMG_SMOOTHER_ADI || k == GMG_SMOOTHER_GSTRI_X || k == GMG_SMOOTHER_GSADI;
}
bool uses_y_lines(int k) {
    return k == GMG_SMOOTHER_TRI_Y || k == GMG_SMOOTHER_ADI || k == GMG_SMOOTHER_GSTRI_Y || k == GMG_SMOOTHER_GSADI;
}

template <int DIR, int MODE>
void launch_line(gmg_problem* p, const Lev& L, const LineFactors& f, const double* rhs, double* ybuf,
                 const double* x, const double* z1, double* out, double damp) {
    const int nl = DIR == 0 ? L.ny : L.nx;
    launch_k(k_line<DIR, MODE>, (nl + kLineT - 1) / kLineT, kLineT, 0, p->st, L.grid(), f, rhs, ybuf, x, z1, out, damp);
    KCHECK();
}

template <int DIR, int MODE>
void launch_gstri(gmg_problem* p, const Lev& L, double om, const LineFactors& f, const double* rhs,
                  const double* x, const double* z1, double* out, double damp) {
    const int nmax = std::max(p->lev(p->L).nx, p->lev(p->L).ny);
    with_coef(L, [&](const auto& A) {
        using C = std::decay_t<decltype(A)>;
        launch_k(k_gstri<DIR, MODE, C>, 1, 32, 0, p->st, L.grid(), A, om, f, rhs, x, z1, out, p->linebuf,
                                                   p->linebuf + nmax, damp);
    });
    KCHECK();
}

// One smooth_step (smoother.cpp:389-399) of a non-Jacobi kind, given the
// defect d = A x - g (in DD, which it may overwrite): out = x - damp*C^{-1} d
// with C^{-1} applied as in apply_preconditioner (smoother.cpp:275-386).
void pc_apply(gmg_problem* p, const Lev& L, const gmg_cycle_desc& sp, const SmLev* m, double* d,
              const double* x, double* out) {
    const double damp = sp.smoothing_omega, om = sp.smoother_omega;
    switch (sp.smoother_kind) {
        case GMG_SMOOTHER_GAUSS_SEIDEL:
        case GMG_SMOOTHER_SOR:
            launch_gs_wave(p, L, d, x, out, om, damp);
            return;
        case GMG_SMOOTHER_RICHARDSON: {
            dim3 gr((L.nx + 127) / 128, L.ny);
            launch_k(k_rich_update, gr, 128, 0, p->st, L.grid(), d, x, out, m->rich, damp);
            KCHECK();
            return;
        }
        case GMG_SMOOTHER_ILU0:
            launch_wave(p, L, IluFwdPolicy{m->lw, m->ls, L.pitch}, d, nullptr, L.scr[0], damp);
            with_coef(L, [&](const auto& A) {
                using C = std::decay_t<decltype(A)>;
                launch_wave(p, L, IluBwdPolicy<C>{A, m->dp, L.pitch}, L.scr[0], x, out, damp);
            });
            return;
        case GMG_SMOOTHER_TRI_X:
            launch_line<0, LO_UPDATE>(p, L, m->fx, d, d, x, nullptr, out, damp);
            return;
        case GMG_SMOOTHER_TRI_Y:
            launch_line<1, LO_UPDATE>(p, L, m->fy, d, d, x, nullptr, out, damp);
            return;
        case GMG_SMOOTHER_ADI:
        case GMG_SMOOTHER_GSADI: {
            // z1 = C_x^{-1} d; t = d - A z1; z = z1 + C_y^{-1} t (smoother.cpp:351-361, 375-384)
            double* z1 = L.scr[0];
            double* t = L.scr[1];
            const bool gs = sp.smoother_kind == GMG_SMOOTHER_GSADI;
            if (gs)
                launch_gstri<0, LO_Z>(p, L, om, m->fx, d, nullptr, nullptr, z1, damp);
            else
                launch_line<0, LO_Z>(p, L, m->fx, d, t, nullptr, nullptr, z1, damp);
            with_coef(L, [&](const auto& A) {
                launch_resid_t(p, L, A, SrcU{z1, L.grid()}, d, t, nullptr, nullptr);
            });
            if (gs)
                launch_gstri<1, LO_SUM_UPDATE>(p, L, om, m->fy, t, x, z1, out, damp);
            else
                launch_line<1, LO_SUM_UPDATE>(p, L, m->fy, t, t, x, z1, out, damp);
            return;
        }
        case GMG_SMOOTHER_GSTRI_X:
            launch_gstri<0, LO_UPDATE>(p, L, om, m->fx, d, x, nullptr, out, damp);
            return;
        case GMG_SMOOTHER_GSTRI_Y:
            launch_gstri<1, LO_UPDATE>(p, L, om, m->fy, d, x, nullptr, out, damp);
            return;
        default:
            throw GmgError{GMG_ERR_LOGIC, "smooth: kind has no preconditioner kernel"};
    }
}

// `steps` smooth_steps of a non-Jacobi kind from source s (a non-u start is
// materialised in bufA; outputs then alternate). Uses DD as defect scratch.
double* pc_steps(gmg_problem* p, const Lev& L, int steps, SmoothSrc s, const double* g, double* bufA,
                 double* bufB, const gmg_cycle_desc& sp, const SmLev* m) {
    if (steps == 0) {
        launch_smooth(p, L, 0, s, g, bufA, sp.smoothing_omega);
        return bufA;
    }
    double* d = L.buf[DD];
    const double* x;
    double* out;
    if (s.kind == S_U) {  // x0 = u in place
        launch_defect_src(p, L, s, g, d, nullptr);
        x = s.u;
        out = (bufA != s.u) ? bufA : bufB;
    } else {  // materialise x0 in bufA (never the buffer a source reads)
        launch_defect_src(p, L, s, g, d, bufA);
        x = bufA;
        out = bufB;
    }
    for (int k = 0; k < steps; ++k) {
        pc_apply(p, L, sp, m, d, x, out);
        if (k + 1 == steps) break;
        SmoothSrc n;
        n.kind = S_U;
        n.u = out;
        launch_defect_src(p, L, n, g, d, nullptr);
        x = out;
        out = (out == bufA) ? bufB : bufA;
    }
    return out;
}

void launch_restrict(gmg_problem* p, int fine_level, const double* f, double* c) {
    const Lev& F = p->lev(fine_level);
    const Lev& C = p->lev(fine_level - 1);
    dim3 b(32, 8), gr((C.nx + 31) / 32, (C.ny + 7) / 8);
    prof_tag("restrict", fine_level, 10.0 * (double)F.n());
    launch_k(k_restrict_simple, gr, b, 0, p->st, F.grid(), f, C.grid(), C.rw, c);
    KCHECK();
}

void launch_coarse(gmg_problem* p, const double* g, double* x) {
    const Lev& L = p->lev(1);
    prof_tag("coarse_solve", 1, 16.0 * (double)L.n());
    launch_k(k_coarse_chol, 1, 32, 0, p->st, p->band, p->cn, p->cbw, L.grid(), g, x, p->cscr);
    KCHECK();
}

void norm_sum(gmg_problem* p, const Lev& L, const double* v, double* out, int mode) {
    seqsum(p, NormTerms{v, L.grid(), 1.0 / L.nx}, L.n(), out, mode);
}

// ---------------------------------------------------------------------------
// row-slab transport: halo rows, gathers, the exact-sum handoff
// ---------------------------------------------------------------------------
NcclApi& nccl() {
    static NcclApi a;
    static std::once_flag once;
    std::call_once(once, [] {
        void* h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
        if (h) {
            a.getUniqueId = reinterpret_cast<decltype(a.getUniqueId)>(dlsym(h, "ncclGetUniqueId"));
            a.commInitRank = reinterpret_cast<decltype(a.commInitRank)>(dlsym(h, "ncclCommInitRank"));
            a.commDestroy = reinterpret_cast<decltype(a.commDestroy)>(dlsym(h, "ncclCommDestroy"));
            a.send = reinterpret_cast<decltype(a.send)>(dlsym(h, "ncclSend"));
            a.recv = reinterpret_cast<decltype(a.recv)>(dlsym(h, "ncclRecv"));
            a.bcast = reinterpret_cast<decltype(a.bcast)>(dlsym(h, "ncclBroadcast"));
            a.allGather = reinterpret_cast<decltype(a.allGather)>(dlsym(h, "ncclAllGather"));
            a.groupStart = reinterpret_cast<decltype(a.groupStart)>(dlsym(h, "ncclGroupStart"));
            a.groupEnd = reinterpret_cast<decltype(a.groupEnd)>(dlsym(h, "ncclGroupEnd"));
            a.errStr = reinterpret_cast<decltype(a.errStr)>(dlsym(h, "ncclGetErrorString"));
        }
    });
    if (!a.send || !a.recv || !a.bcast || !a.allGather || !a.groupStart || !a.groupEnd || !a.commInitRank)
        throw GmgError{GMG_ERR_UNSUPPORTED, "row-slab mode needs libnccl.so.2"};
    return a;
}
#define NC(x)                                                                                   \
    do {                                                                                        \
        const int r_ = (x);                                                                     \
        if (r_ != 0) throw GmgError{GMG_ERR_CUDA, std::string("nccl: ") + nccl().errStr(r_)};   \
    } while (0)

// buffer ids: level buffers U0..DD, and the finest level's x ping-pong and b
enum BufId { B_X0 = 10, B_X1 = 11, B_B = 12 };
double* bufptr(gmg_problem* q, int l, int id) {
    if (id == B_X0) return q->X[0];
    if (id == B_X1) return q->X[1];
    if (id == B_B) return q->B;
    return q->lev(l).buf[id];
}

// rows [a, b) of a level-l buffer, as whole pitched rows
struct RowSpan {
    double* p;
    size_t count;
};
RowSpan rows_of(gmg_problem* q, int l, int id, int a, int b) {
    const Lev& L = q->lev(l);
    return RowSpan{bufptr(q, l, id) + (long long)a * L.pitch, (size_t)std::max(0, b - a) * (size_t)L.pitch};
}

// Refresh `rows` halo rows on both sides of every slab boundary of level l.
void dist_halo(const std::vector<gmg_problem*>& S, DistCtx& D, int l, int id, int rows) {
    const auto& w0 = D.w0[l - 1];
    const auto& w1 = D.w1[l - 1];
    cudaStream_t st = S[0]->st;
    if (D.local) {
        for (int r = 0; r + 1 < D.world; ++r) {
            const int e = w1[r];  // == w0[r + 1]
            const RowSpan up = rows_of(S[r], l, id, e - rows, e), upd = rows_of(S[r + 1], l, id, e - rows, e);
            CK(cudaMemcpyAsync(upd.p, up.p, up.count * sizeof(double), cudaMemcpyDeviceToDevice, st));
            if (g_debug_sync) dbg_sync(__LINE__);
            const RowSpan dn = rows_of(S[r + 1], l, id, e, e + rows), dnd = rows_of(S[r], l, id, e, e + rows);
            CK(cudaMemcpyAsync(dnd.p, dn.p, dn.count * sizeof(double), cudaMemcpyDeviceToDevice, st));
            if (g_debug_sync) dbg_sync(__LINE__);
        }
        return;
    }
    gmg_problem* q = S[0];
    const int r = q->rank;
    NcclApi& n = nccl();
    NC(n.groupStart());
    if (r > 0) {
        const RowSpan mine = rows_of(q, l, id, w0[r], w0[r] + rows), theirs = rows_of(q, l, id, w0[r] - rows, w0[r]);
        NC(n.send(mine.p, mine.count, kNcclFloat64, r - 1, D.comm, st));
        NC(n.recv(theirs.p, theirs.count, kNcclFloat64, r - 1, D.comm, st));
    }
    if (r + 1 < D.world) {
        const RowSpan mine = rows_of(q, l, id, w1[r] - rows, w1[r]), theirs = rows_of(q, l, id, w1[r], w1[r] + rows);
        NC(n.send(mine.p, mine.count, kNcclFloat64, r + 1, D.comm, st));
        NC(n.recv(theirs.p, theirs.count, kNcclFloat64, r + 1, D.comm, st));
    }
    NC(n.groupEnd());
}

// Every rank's rows [a[r], b[r]) of a level-l buffer to every rank.
void dist_gather(const std::vector<gmg_problem*>& S, DistCtx& D, int l, int id, const std::vector<int>& a,
                 const std::vector<int>& b) {
    cudaStream_t st = S[0]->st;
    if (D.local) {
        for (int r = 0; r < D.world; ++r)
            for (int t = 0; t < D.world; ++t)
                if (t != r) {
                    const RowSpan src = rows_of(S[r], l, id, a[r], b[r]), dst = rows_of(S[t], l, id, a[r], b[r]);
                    if (src.count)
                        CK(cudaMemcpyAsync(dst.p, src.p, src.count * sizeof(double), cudaMemcpyDeviceToDevice, st));
                    if (g_debug_sync) dbg_sync(__LINE__);
                }
        return;
    }
    NcclApi& n = nccl();
    NC(n.groupStart());
    for (int r = 0; r < D.world; ++r) {
        const RowSpan sp = rows_of(S[0], l, id, a[r], b[r]);
        if (sp.count) NC(n.bcast(sp.p, sp.p, sp.count, kNcclFloat64, r, D.comm, st));
    }
    NC(n.groupEnd());
}

// The coarse rows that rank r's slab of sharded level l restricts into (the
// centre fine row 2Q+1 lies in the slab): [w0/2, w1/2).
void threshold_rows(const DistCtx& D, int l, std::vector<int>& a, std::vector<int>& b) {
    a.resize(D.world);
    b.resize(D.world);
    for (int r = 0; r < D.world; ++r) {
        a[r] = D.w0[l - 1][r] / 2;
        b[r] = D.w1[l - 1][r] / 2;
    }
}

__global__ void k_nz_to_d(const int* __restrict__ nz, double* __restrict__ out) {
    pdl_wait();  // programmatic dependent launch: inputs of the previous kernel are complete
    pdl_trigger(); out[0] = nz[0] ? 1.0 : 0.0; }

// From the gathered per-rank approximate totals g[r*8 + k] (k < NS; k == NS:
// nz flag): pre[k] = sum over ranks below `rank` (seeds the walk), nz = OR,
// and for the fast mode the rank-ordered total.
__global__ void k_dist_prefix(const double* __restrict__ g, int rank, int world, int ns, int with_nz,
                              double* __restrict__ pre, int* __restrict__ nz, double* __restrict__ total) {
    pdl_wait();  // programmatic dependent launch: inputs of the previous kernel are complete
    pdl_trigger();
    if (threadIdx.x != 0) return;
    for (int k = 0; k < ns; ++k) {
        double a = 0.0, t = 0.0;
        for (int r = 0; r < world; ++r) {
            if (r < rank) a += g[r * 8 + k];
            t += g[r * 8 + k];
        }
        pre[k] = a;
        if (total) total[k] = t;
    }
    if (with_nz) {
        int any = 0;
        for (int r = 0; r < world; ++r) any |= g[r * 8 + ns] != 0.0;
        *nz = any;
    }
}

// A reduction over a sharded level: slab r sums the terms of its own rows.
// EXACT: walks run per slab from approximate rank prefixes, then the chains run
// in rank order, each starting from the exact state its predecessor ended in,
// and the last rank's result is broadcast: the reference's k order exactly.
// `make(q)` returns {term generator, term count} for slab q.
template <class MakeTG>
void dist_sum(const std::vector<gmg_problem*>& S, DistCtx* D, MakeTG make, int out_off, int mode, bool with_nz) {
    using TG = decltype(make(S[0]).first);
    constexpr int NS = TG::NS;
    if (!D) {  // a replicated level: every slab sums its own (identical) copy
        for (auto* q : S) {
            auto tn = make(q);
            seqsum(q, tn.first, tn.second, q->sums + out_off, mode);
        }
        return;
    }
    cudaStream_t st = S[0]->st;
    // 1. approximate totals (and the nz flag) of every slab, gathered everywhere
    for (auto* q : S) {
        auto tn = make(q);
        seqsum_fast(q, tn.first, tn.second, q->dscr, nullptr);
        if (with_nz) launch_k(k_nz_to_d, 1, 1, 0, st, q->nz_cur, q->dscr + NS);
    }
    KCHECK();
    if (D->local) {
        for (auto* q : S)
            for (auto* t : S)
                CK(cudaMemcpyAsync(t->dscr + 32 + 8 * q->rank, q->dscr, 8 * sizeof(double), cudaMemcpyDeviceToDevice,
                                   st));
    } else {
        NC(nccl().allGather(S[0]->dscr, S[0]->dscr + 32, 8, kNcclFloat64, D->comm, st));
    }
    for (auto* q : S)
        launch_k(k_dist_prefix, 1, 32, 0, st, q->dscr + 32, q->rank, D->world, NS, with_nz ? 1 : 0, q->dscr + 8, q->nz_cur,
                                        mode == GMG_REDUCE_FAST ? q->sums + out_off : nullptr);
    KCHECK();
    if (mode == GMG_REDUCE_FAST) return;
    // 2. walks (independent), 3. chains in rank order, 4. broadcast of the total
    for (auto* q : S) {
        auto tn = make(q);
        seqsum_walk(q, tn.first, tn.second, q->dscr + 8);
    }
    if (D->local) {
        for (size_t r = 0; r < S.size(); ++r) {
            auto tn = make(S[r]);
            seqsum_chain(S[r], tn.first, tn.second, S[r]->sums + out_off, r ? S[r - 1]->sums + out_off : nullptr);
        }
        for (size_t r = 0; r + 1 < S.size(); ++r)
            CK(cudaMemcpyAsync(S[r]->sums + out_off, S.back()->sums + out_off, NS * sizeof(double),
                               cudaMemcpyDeviceToDevice, st));
        return;
    }
    gmg_problem* q = S[0];
    const int r = q->rank;
    NcclApi& n = nccl();
    if (r > 0) NC(n.recv(q->dscr + 16, NS, kNcclFloat64, r - 1, D->comm, st));
    auto tn = make(q);
    seqsum_chain(q, tn.first, tn.second, q->sums + out_off, r ? q->dscr + 16 : nullptr);
    if (r + 1 < D->world) NC(n.send(q->sums + out_off, NS, kNcclFloat64, r + 1, D->comm, st));
    NC(n.bcast(q->sums + out_off, q->sums + out_off, NS, kNcclFloat64, D->world - 1, D->comm, st));
}

// ---------------------------------------------------------------------------
// cycle driver (recorded into a CUDA graph)
// ---------------------------------------------------------------------------
// A smoothing start in buffer ids (SmoothSrc with per-slab pointers).
struct SrcId {
    Start kind = S_ZERO;
    int u = -1;   // level-l buffer (S_U, S_CORRECT)
    int uc = -1;  // level-(l-1) buffer (S_PROLONG, S_CORRECT)
    bool adaptive = false;
};

struct Driver {
    std::vector<gmg_problem*> S;  // the slabs this process drives, in rank order (one without row slabs)
    gmg_cycle_desc sp;
    const SmSetup* sm = nullptr;  // setup_smoothers products (null for jacobi / GS / SOR)

    gmg_problem* p() const { return S[0]; }
    DistCtx* D() const { return S[0]->dist.get(); }
    bool sharded(int l) const { return D() && l >= D()->Ls; }
    void halo(int l, int id, int rows) {
        if (sharded(l)) dist_halo(S, *D(), l, id, rows);
    }
    // after a restriction from sharded level l into replicated level l-1
    void gather_threshold(int l, int id_coarse) {
        if (!sharded(l) || sharded(l - 1)) return;
        std::vector<int> a, b;
        threshold_rows(*D(), l, a, b);
        dist_gather(S, *D(), l - 1, id_coarse, a, b);
    }
    SmoothSrc resolve(gmg_problem* q, int l, const SrcId& s) const {
        SmoothSrc r;
        r.kind = s.kind;
        if (s.u >= 0) r.u = bufptr(q, l, s.u);
        if (s.uc >= 0) r.uc = bufptr(q, l - 1, s.uc);
        r.om = s.adaptive ? OmegaSrc{q->sums, q->nz_cur, 0.0, q->status}
                          : OmegaSrc{nullptr, nullptr, sp.correction_omega, q->status};
        return r;
    }

    // smooth_step x `steps` with the configured preconditioner (setup_smoothers);
    // outputs alternate a, b. Returns the id of the result.
    int smooth(int l, int steps, SrcId s, int g, int a, int b) {
        if (sp.smoother_kind != GMG_SMOOTHER_JACOBI) {
            if (D()) throw GmgError{GMG_ERR_UNSUPPORTED, "row slabs: only the jacobi smoother is sharded"};
            gmg_problem* q = p();
            const Lev& L = q->lev(l);
            const double* r = pc_steps(q, L, steps, resolve(q, l, s), bufptr(q, l, g), bufptr(q, l, a),
                                       bufptr(q, l, b), sp, sm ? &sm->lev[l - 1] : nullptr);
            return r == bufptr(q, l, a) ? a : b;
        }
        if (sharded(l)) {
            const int H = D()->H;
            halo(l, g, H);
            if (s.u >= 0) halo(l, s.u, H);
            if (s.uc >= 0) halo(l - 1, s.uc, H);
        }
        int dst = a;
        int left = steps;
        bool first = true;
        while (first || left > 0) {
            const int M = std::min(left, kMaxFuse);
            for (auto* q : S)
                launch_smooth(q, q->lev(l), M, resolve(q, l, s), bufptr(q, l, g), bufptr(q, l, dst),
                              sp.smoothing_omega);
            left -= M;
            first = false;
            s = SrcId{};
            s.kind = S_U;
            s.u = dst;
            if (left > 0) {
                halo(l, dst, D() ? D()->H : 0);
                dst = (dst == a) ? b : a;
            }
        }
        return dst;
    }

    // levels <= kVTop in one CTA (k_vsmall): Jacobi V recursion from a zero or
    // prolongated start, every slab replicated (none of these levels is sharded)
    bool fused_small(int l, const SrcId& s) const {
        if (l > kVTop || sp.smoother_kind != GMG_SMOOTHER_JACOBI || sp.cycle == GMG_CYCLE_W) return false;
        if (s.kind != S_ZERO && s.kind != S_PROLONG) return false;
        if (sharded(l)) return false;
        return vsmall_smem(l) <= kVSmemMax;
    }
    size_t vsmall_smem(int l) const {
        size_t nd = 0;
        for (int q = 1; q <= l; ++q) nd += 3 * (size_t)p()->lev(q).n();
        nd += 2 * (size_t)p()->lev(l).n();
        return nd * sizeof(double);
    }
    void launch_vsmall(gmg_problem* q, int l, const SrcId& s, int g) {
        VParams V{};
        int off = 0;
        for (int k = 1; k <= l; ++k) {
            const Lev& L = q->lev(k);
            VLev& v = V.lv[k];
            v.nx = L.nx;
            v.ny = L.ny;
            v.pitch = L.pitch;
            v.kind = L.kind;
            v.per = L.per;
            v.cc = L.cconst;
            v.cr = L.crow;
            v.cf = L.cfield;
            v.ca = L.caxes;
            v.tx = L.tx;
            v.ty = L.ty;
            v.rw = L.rw;
            v.off = off;
            off += 3 * L.nx * L.ny;
        }
        V.toff = off;
        V.top = l;
        V.pre = sp.pre_steps;
        V.post = sp.post_steps;
        V.adaptive = sp.adaptive_correction != 0;
        V.direct = (unsigned long long)q->lev(1).n() <= sp.coarse_direct_max_neq;
        V.cn = q->cn;
        V.cbw = q->cbw;
        V.damp = sp.smoothing_omega;
        V.corr_omega = sp.correction_omega;
        V.band = q->band;
        V.g_top = bufptr(q, l, g);
        V.uc = s.kind == S_PROLONG ? bufptr(q, l - 1, s.uc) : nullptr;
        V.out = q->lev(l).buf[U0];
        V.status = q->status;
        set_smem(k_vsmall, kVSmemMax);
        prof_tag("vsmall(V below)", l, 0.0);
        launch_k(k_vsmall, 1, kVThreads, vsmall_smem(l), q->st, V);
        KCHECK();
    }

    // gmg::mg_cycle (cycle.cpp:69-100) on level l from start s with rhs g.
    int visit(int l, SrcId s, int g) {
        if (fused_small(l, s)) {
            for (auto* q : S) launch_vsmall(q, l, s, g);
            return U0;
        }
        const int u_in = s.kind == S_U ? s.u : -1;
        const int a = (u_in == U0) ? U1 : U0;
        const int b = (a == U0) ? U1 : U0;
        if (l == 1) {
            // coarse_solve (cycle.cpp:57-65)
            if ((unsigned long long)p()->lev(1).n() <= sp.coarse_direct_max_neq) {
                for (auto* q : S) launch_coarse(q, bufptr(q, 1, g), q->lev(1).buf[U0]);
                return U0;
            }
            return smooth(1, std::max(1, sp.pre_steps + sp.post_steps), s, g, a, b);
        }
        const int u = smooth(l, sp.pre_steps, s, g, a, b);
        const int other = (u == U0) ? U1 : U0;
        const bool adaptive = sp.adaptive_correction != 0;
        // the post-smoothing start u + w*P uc reads u within the halo; the residual needs 2 rows
        halo(l, u, D() ? D()->H : 0);
        for (auto* q : S) {
            Lev& L = q->lev(l);
            launch_resid(q, L, L.buf[u], nullptr, bufptr(q, l, g), adaptive ? L.buf[DD] : nullptr, nullptr,
                         q->lev(l - 1).buf[GRHS]);
        }
        gather_threshold(l, GRHS);
        SrcId z;
        int uc = visit(l - 1, z, GRHS);
        if (sp.cycle == GMG_CYCLE_W) {
            SrcId w;
            w.kind = S_U;
            w.u = uc;
            uc = visit(l - 1, w, GRHS);
        }
        if (sharded(l - 1)) halo(l - 1, uc, D()->H);
        SrcId cs;
        cs.kind = S_CORRECT;
        cs.u = u;
        cs.uc = uc;
        cs.adaptive = adaptive;
        if (adaptive) omega_sums_d(l, uc);
        return smooth(l, sp.post_steps, cs, g, other, u);
    }

    // adaptive_omega sums (cycle.cpp:40-51) for corr = P uc over each slab's rows
    void omega_sums_d(int l, int uc) {
        for (auto* q : S) {
            Lev& L = q->lev(l);
            // this visit's flag slot (zeroed at the cycle start); beyond the slots, a memset
            if (q->nz_next < gmg_problem::kNzSlots) {
                q->nz_cur = q->nz_slots + q->nz_next++;
            } else {
                q->nz_cur = q->nz;
                CK(cudaMemsetAsync(q->nz, 0, sizeof(int), q->st));
            }
            const int seg = seg_rows(L.nx, L.rows());
            dim3 grid((L.nx + (kTW - 2) - 1) / (kTW - 2), (L.rows() + seg - 1) / seg);
            SrcProlong src{prolong_from(q, l - 1, q->lev(l - 1).buf[uc]), L.nx, L.ny, 0.0};
            double* T0 = q->T;
            double* T1 = q->T + q->lev(q->L).n();
            if (L.strips()) {
                with_coef_big(L, [&](const auto& A) {
                    using C = std::decay_t<decltype(A)>;
                    set_smem(k_omega4<C>, omega4_smem());
                    const int strips = (L.nx + 123) / 124;
                    dim3 g4((strips + kS4W - 1) / kS4W, (L.rows() + seg - 1) / seg);
                    prof_tag("omega terms", l, 26.0 * (double)L.nx * L.rows());
                    launch_k(k_omega4<C>, g4, kS4W * 32, omega4_smem(), q->st, L.grid(), A, src.P, L.buf[DD], T0, T1,
                             q->nz_cur, seg);
                });
            } else {
                with_coef(L, [&](const auto& A) {
                    using C = std::decay_t<decltype(A)>;
                    prof_tag("omega terms", l, 26.0 * (double)L.nx * L.rows());
                    launch_k(k_omega_terms<kTW, 2, C>, grid, kTW, 0, q->st, L.grid(), A, src, L.buf[DD], T0, T1,
                             q->nz_cur, seg);
                });
            }
            KCHECK();
        }
        g_cur_level = l;
        dist_sum(S, sharded(l) ? D() : nullptr, [&](gmg_problem* q) {
            const Lev& L = q->lev(l);
            const long long o = (long long)L.w0 * L.nx;
            return std::make_pair(ArrTerms{q->T + o, q->T + q->lev(q->L).n() + o}, (long long)L.rows() * L.nx);
        }, 0, sp.reduction, true);
    }

    // exact-order ||v||^2 of a level-l buffer over the owned rows -> sums[off]
    void norm_d(int l, int id, int off) {
        g_cur_level = l;
        dist_sum(S, sharded(l) ? D() : nullptr, [&](gmg_problem* q) {
            const Lev& L = q->lev(l);
            Grid gv{L.nx, L.rows(), L.pitch, 0, L.rows()};
            return std::make_pair(NormTerms{bufptr(q, l, id) + (long long)L.w0 * L.pitch, gv, 1.0 / L.nx},
                                  (long long)L.rows() * L.nx);
        }, off, sp.reduction, false);
    }

    // residual of x (+ e) against b on the finest level -> DCAS[L], x0 -> xout, restricted -> DCAS[L-1]
    void final_resid(int xin, int e, int xout, bool restrict_) {
        const int L = p()->L;
        if (sharded(L)) {
            halo(L, xin, 2);
            if (e >= 0) halo(L, e, 2);
        }
        for (auto* q : S) {
            Lev& F = q->lev(L);
            launch_resid(q, F, bufptr(q, L, xin), e >= 0 ? F.buf[e] : nullptr, q->B, F.buf[DCAS], bufptr(q, L, xout),
                         restrict_ ? q->lev(L - 1).buf[DCAS] : nullptr);
        }
        if (restrict_) gather_threshold(L, DCAS);
    }

    // One outer cycle: x_out = cycle(x_in); r = b - A x_out -> DCAS[L]; norm^2 -> sums[2].
    void cycle(int xin, int xout) {
        const int L = p()->L;
        for (auto* q : S) {  // fresh "correction nonzero" slots for this cycle's level visits
            CK(cudaMemsetAsync(q->nz_slots, 0, gmg_problem::kNzSlots * sizeof(int), q->st));
            q->nz_next = 0;
        }
        if (sp.cycle == GMG_CYCLE_F) {
            // fcycle_pass (cycle.cpp:119-142): DCAS[L], DCAS[L-1] are current
            for (int l = L - 1; l >= 2; --l) {
                if (sharded(l)) halo(l, DCAS, 1);
                for (auto* q : S) launch_restrict(q, l, q->lev(l).buf[DCAS], q->lev(l - 1).buf[DCAS]);
                gather_threshold(l, DCAS);
            }
            SrcId z;
            if (L == 1) {
                SrcId s0;
                s0.kind = S_U;
                s0.u = xin;
                const int e = visit_top(s0);
                final_resid(e, -1, xout, false);
            } else {
                int e = visit(1, z, DCAS);
                for (int l = 2; l <= L; ++l) {
                    SrcId s;
                    s.kind = S_PROLONG;
                    s.uc = e;
                    e = visit(l, s, DCAS);
                }
                final_resid(xin, e, xout, true);
            }
        } else {
            SrcId s0;
            s0.kind = S_U;
            s0.u = xin;
            const int e = visit_top(s0);
            final_resid(e, -1, xout, false);
        }
        norm_d(L, DCAS, 2);
    }

    // r0 = b - A x0 -> DCAS[L] (x0 in X[0], complete on every slab), and for the
    // F-cycle its restriction, the first defect cascade seed
    void initial_resid() {
        const int L = p()->L;
        const bool restr = sp.cycle == GMG_CYCLE_F && L >= 2;
        for (auto* q : S) {
            Lev& F = q->lev(L);
            launch_resid(q, F, q->X[0], nullptr, q->B, F.buf[DCAS], nullptr, restr ? q->lev(L - 1).buf[DCAS] : nullptr);
        }
        if (restr) gather_threshold(L, DCAS);
    }

    // visit of the finest level with rhs b (V/W cycles, single level)
    int visit_top(SrcId s0) { return visit(p()->L, s0, B_B); }
};

std::string spec_key(const gmg_cycle_desc& s) {
    char buf[256];
    std::snprintf(buf, sizeof buf, "%d|%d|%d|%d|%a|%d|%a|%a|%llu|%d", s.cycle, s.pre_steps, s.post_steps,
                  s.adaptive_correction, s.correction_omega, s.smoother_kind, s.smoother_omega,
                  s.smoothing_omega, s.coarse_direct_max_neq, s.reduction);
    return buf;
}

const SmSetup* find_smoother(gmg_problem* p, const gmg_cycle_desc& sp);

// the slabs a driver on this handle runs: all virtual ranks of a local cluster, else itself
std::vector<gmg_problem*> driver_slabs(gmg_problem* p) {
    if (p->dist && p->dist->local) return p->dist->slabs;
    return {p};
}

std::array<cudaGraphExec_t, 2>& get_graphs(gmg_problem* p, const gmg_cycle_desc& sp) {
    const std::string key = spec_key(sp);
    auto it = p->graphs.find(key);
    if (it != p->graphs.end()) return it->second;
    std::array<cudaGraphExec_t, 2> ex{};
    for (int par = 0; par < 2; ++par) {
        cudaGraph_t g = nullptr;
        CK(cudaStreamBeginCapture(p->st, cudaStreamCaptureModeThreadLocal));
        try {
            Driver d{driver_slabs(p), sp, find_smoother(p, sp)};
            d.cycle(par == 0 ? B_X0 : B_X1, par == 0 ? B_X1 : B_X0);
        } catch (...) {
            cudaStreamEndCapture(p->st, &g);
            if (g) cudaGraphDestroy(g);
            throw;
        }
        CK(cudaStreamEndCapture(p->st, &g));
        CK(cudaGraphInstantiate(&ex[par], g, 0));
        CK(cudaGraphDestroy(g));
    }
    return p->graphs.emplace(key, ex).first->second;
}

// smoother admissibility, smoother.cpp:51-69 (setup_smoothers runs first in solve)
void check_smoother(const gmg_cycle_desc& sp) {
    const double w = sp.smoother_omega;
    switch (sp.smoother_kind) {
        case GMG_SMOOTHER_RICHARDSON:
        case GMG_SMOOTHER_JACOBI:
        case GMG_SMOOTHER_ILU0:
            if (!(w > 0.0)) throw std::invalid_argument("smoother_omega: must be > 0");
            break;
        case GMG_SMOOTHER_GAUSS_SEIDEL:
        case GMG_SMOOTHER_SOR:
            if (!(w > 0.0 && w < 2.0))
                throw std::invalid_argument("smoother_omega: must be in (0, 2) for gauss_seidel/sor");
            break;
        case GMG_SMOOTHER_TRI_X:
        case GMG_SMOOTHER_TRI_Y:
        case GMG_SMOOTHER_ADI:
        case GMG_SMOOTHER_GSTRI_X:
        case GMG_SMOOTHER_GSTRI_Y:
        case GMG_SMOOTHER_GSADI:
            if (!(w > 0.0 && w <= 1.0))
                throw std::invalid_argument("smoother_omega: must be in (0, 1] for line smoothers");
            break;
        default:
            throw std::invalid_argument("smoother: unknown kind");
    }
}

// Periodic (polar) levels define the pointwise smoothers only: the lexicographic
// and line sweeps would need wrap-around recurrences.
void check_periodic_kind(const gmg_problem* p, int kind) {
    if (p->lv[0].per && kind != GMG_SMOOTHER_JACOBI && kind != GMG_SMOOTHER_RICHARDSON)
        throw std::invalid_argument("smoother: periodic (polar) grids support jacobi and richardson only");
}

// checks the reference performs inside mg_cycle / smooth_step (cycle.cpp:75-76, smoother.cpp:391)
void check_cycle(const gmg_problem* p, const gmg_cycle_desc& sp) {
    if (sp.pre_steps < 0 || sp.post_steps < 0 || sp.pre_steps + sp.post_steps < 1)
        throw std::invalid_argument("pre_steps/post_steps: at least one smoothing step per visit");
    const bool smooths = p->L > 1 || (unsigned long long)p->lv[0].n() > sp.coarse_direct_max_neq;
    if (smooths && !(sp.smoothing_omega > 0.0)) throw std::invalid_argument("omega: damping must be > 0");
    if (sp.cycle < 0 || sp.cycle > 2) throw std::invalid_argument("cycle: must be one of V, W, F");
}

// Transfers of pageable host vectors (the C++ shim passes std::vector storage, and
// gmg::solve's b and x are such vectors): staged through a small pinned ring by a few
// host threads, so the host copy of one chunk of rows overlaps the DMA of the previous
// ones. The CUDA runtime's own pageable path runs at about a fifth of the link rate.
// Pinned or registered buffers, and small ones, go straight to the copy engine.
bool host_pageable(const void* h) {
    cudaPointerAttributes a{};
    if (cudaPointerGetAttributes(&a, h) != cudaSuccess) {
        cudaGetLastError();
        return true;
    }
    return a.type == cudaMemoryTypeUnregistered;
}

// The ring, allocated on first use. A host that cannot pin 64 MB (locked-memory limits) keeps
// the runtime's pageable copy: slower, never wrong.
bool stage_ready(gmg_problem* p) {
    if (p->stage) return true;
    if (p->stage_failed) return false;
    if (cudaHostAlloc(&p->stage, (size_t)kStageThreads * kStageSlots * kStageBytes, cudaHostAllocDefault) !=
        cudaSuccess) {
        cudaGetLastError();
        p->stage = nullptr;
        p->stage_failed = true;
        return false;
    }
    for (auto& e : p->stage_ev) CK(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
    return true;
}

void staged_rows(gmg_problem* p, const Lev& L, double* dev, double* host, bool to_device) {
    const size_t rowb = (size_t)L.nx * sizeof(double);
    const int rows_per = (int)std::max<size_t>(1, kStageBytes / rowb);
    const int nchunks = (L.ny + rows_per - 1) / rows_per;
    const int T = std::min(g_stage_threads, nchunks);
    std::exception_ptr err[kStageThreads];
    auto work = [&](int t) {
        try {
            CK(cudaSetDevice(p->device));
            auto slot = [&](int s) { return p->stage + ((size_t)t * kStageSlots + s) * kStageBytes; };
            auto ev = [&](int s) { return p->stage_ev[t * kStageSlots + s]; };
            auto rows0 = [&](int k) { return (t + k * T) * rows_per; };
            auto nrows = [&](int k) { return std::min(rows_per, L.ny - rows0(k)); };
            const int mine = (nchunks - t + T - 1) / T;
            if (to_device) {
                for (int k = 0; k < mine; ++k) {
                    const int s = k % kStageSlots;
                    CK(cudaEventSynchronize(ev(s)));  // the DMA that last read this slot (any earlier call too)
                    std::memcpy(slot(s), host + (size_t)rows0(k) * L.nx, nrows(k) * rowb);
                    CK(cudaMemcpy2DAsync(dev + (size_t)rows0(k) * L.pitch, L.pitch * sizeof(double), slot(s), rowb, rowb,
                                         nrows(k), cudaMemcpyHostToDevice, p->st));
                    CK(cudaEventRecord(ev(s), p->st));
                }
            } else {
                auto issue = [&](int k) {
                    const int s = k % kStageSlots;
                    CK(cudaMemcpy2DAsync(slot(s), rowb, dev + (size_t)rows0(k) * L.pitch, L.pitch * sizeof(double), rowb,
                                         nrows(k), cudaMemcpyDeviceToHost, p->st));
                    CK(cudaEventRecord(ev(s), p->st));
                };
                for (int k = 0; k < std::min(mine, kStageSlots); ++k) issue(k);
                for (int k = 0; k < mine; ++k) {
                    const int s = k % kStageSlots;
                    CK(cudaEventSynchronize(ev(s)));
                    std::memcpy(host + (size_t)rows0(k) * L.nx, slot(s), nrows(k) * rowb);
                    if (k + kStageSlots < mine) issue(k + kStageSlots);
                }
            }
        } catch (...) {
            err[t] = std::current_exception();
        }
    };
    std::vector<std::thread> th;
    for (int t = 1; t < T; ++t) th.emplace_back(work, t);
    work(0);
    for (auto& x : th) x.join();
    for (int t = 0; t < T; ++t)
        if (err[t]) std::rethrow_exception(err[t]);
}

bool stage_this(gmg_problem* p, const Lev& L, const void* host, cudaMemcpyKind kind) {
    return (kind == cudaMemcpyHostToDevice || kind == cudaMemcpyDeviceToHost) && !g_no_stage &&
           (size_t)L.nx * L.ny * sizeof(double) >= kStageMin && (size_t)L.nx * sizeof(double) <= kStageBytes &&
           host_pageable(host) && stage_ready(p);
}

void upload(gmg_problem* p, const Lev& L, double* dst, const double* src, cudaMemcpyKind kind) {
    if (stage_this(p, L, src, kind)) {
        staged_rows(p, L, dst, const_cast<double*>(src), true);
    } else {
        CK(cudaMemcpy2DAsync(dst, L.pitch * sizeof(double), src, L.nx * sizeof(double), L.nx * sizeof(double),
                             L.ny, kind, p->st));
    }
    if (g_debug_sync) dbg_sync(__LINE__);
}
void download(gmg_problem* p, const Lev& L, double* dst, const double* src, cudaMemcpyKind kind) {
    if (stage_this(p, L, dst, kind)) {
        staged_rows(p, L, const_cast<double*>(src), dst, false);
    } else {
        CK(cudaMemcpy2DAsync(dst, L.nx * sizeof(double), src, L.pitch * sizeof(double), L.nx * sizeof(double),
                             L.ny, kind, p->st));
    }
    if (g_debug_sync) dbg_sync(__LINE__);
}

double fetch_scalar(gmg_problem* p, const double* dev) {
    CK(cudaMemcpyAsync(p->hostbuf, dev, sizeof(double), cudaMemcpyDeviceToHost, p->st));
    if (g_debug_sync) dbg_sync(__LINE__);
    CK(cudaStreamSynchronize(p->st));
    return p->hostbuf[0];
}

int fetch_status(gmg_problem* p) {
    int s = 0;
    CK(cudaMemcpyAsync(&s, p->status, sizeof(int), cudaMemcpyDeviceToHost, p->st));
    if (g_debug_sync) dbg_sync(__LINE__);
    CK(cudaStreamSynchronize(p->st));
    return s;
}

// The reference's five operator arrays of a level (c, w, e, s, n), rebuilt
// from the device classes: CONST/ROWX with their exact zeros toward the
// boundary, FIELD downloaded.
void host_coefs(gmg_problem* p, const Lev& L, std::vector<double> (&a)[5]) {
    const size_t N = (size_t)L.n();
    for (auto& v : a) v.assign(N, 0.0);
    if (L.kind == 3) {  // the AXES expressions (common.cuh CoefAxes), on the host
        const gmg_host::AxisTables& T = L.axt;
        for (int j = 0; j < L.ny; ++j)
            for (int i = 0; i < L.nx; ++i) {
                const size_t k = (size_t)j * L.nx + i;
                const double ce = (T.ae[i] * T.my[j]) / T.he[i], cw = (T.aw[i] * T.my[j]) / T.hw[i];
                const double cn = (T.bn[j] * T.mx[i]) / T.hn[j], cs = (T.bs[j] * T.mx[i]) / T.hs[j];
                a[0][k] = ((ce + cw) + cn) + cs;
                a[1][k] = i > 0 ? -cw : 0.0;
                a[2][k] = i + 1 < L.nx ? -ce : 0.0;
                a[3][k] = j > 0 ? -cs : 0.0;
                a[4][k] = j + 1 < L.ny ? -cn : 0.0;
            }
        return;
    }
    if (L.kind == 2) {
        for (int q = 0; q < 5; ++q)
            download(p, L, a[q].data(), L.coefmem + q * L.elems + L.off0, cudaMemcpyDeviceToHost);
        CK(cudaStreamSynchronize(p->st));
        return;
    }
    std::vector<double> row[5];
    if (L.kind == 1) {
        for (int q = 0; q < 5; ++q) {
            row[q].resize(L.nx);
            CK(cudaMemcpy(row[q].data(), L.coefmem + q * L.nx, L.nx * sizeof(double), cudaMemcpyDeviceToHost));
        }
    } else {
        const double v[5] = {L.cconst.c, L.cconst.w, L.cconst.e, L.cconst.s, L.cconst.n};
        for (int q = 0; q < 5; ++q) row[q].assign(L.nx, v[q]);
    }
    for (int j = 0; j < L.ny; ++j)
        for (int i = 0; i < L.nx; ++i) {
            const size_t k = (size_t)j * L.nx + i;
            a[0][k] = row[0][i];
            a[1][k] = (L.kind == 1 || i > 0) ? row[1][i] : 0.0;
            a[2][k] = (L.kind == 1 || i + 1 < L.nx) ? row[2][i] : 0.0;
            a[3][k] = j > 0 ? row[3][i] : 0.0;
            a[4][k] = j + 1 < L.ny ? row[4][i] : 0.0;
        }
}

void ensure_scratch(gmg_problem* p, Lev& L) {
    if (L.scrmem) return;
    CK(dmalloc(&L.scrmem, 2 * L.elems * sizeof(double)));
    CK(cudaMemsetAsync(L.scrmem, 0, 2 * L.elems * sizeof(double), p->st));
    if (g_debug_sync) dbg_sync(__LINE__);
    L.scr[0] = L.scrmem + L.off0;
    L.scr[1] = L.scrmem + L.elems + L.off0;
}

// richardson setup (smoother.cpp:240-251): power_apply_A(op, 20) (:212-227)
// from mt19937(0x2d5a11) uniform(-1,1), exact-order norms, then the clamp.
double richardson_omega(gmg_problem* p, Lev& L, double omega) {
    std::vector<double> x0((size_t)L.n());
    std::mt19937 rng(0x2d5a11u);
    std::uniform_real_distribution<double> dist(-1.0, 1.0);
    for (double& v : x0) v = dist(rng);
    double* xa = L.buf[U0];
    double* ya = L.buf[U1];
    upload(p, L, xa, x0.data(), cudaMemcpyHostToDevice);
    double lambda = 0.0;
    for (int t = 0; t < 20; ++t) {
        with_coef(L, [&](const auto& A) {
            dim3 b(32, 8), gr((L.nx + 31) / 32, (L.ny + 7) / 8);
            launch_k(k_apply_simple<std::decay_t<decltype(A)>>, gr, b, 0, p->st, L.grid(), A, xa, ya);
        });
        KCHECK();
        norm_sum(p, L, ya, p->sums + 3, GMG_REDUCE_EXACT);
        lambda = std::sqrt(fetch_scalar(p, p->sums + 3));
        if (lambda == 0.0) break;
        launch_k(k_div_scalar, dim3((L.nx + 127) / 128, L.ny), 128, 0, p->st, L.grid(), ya, lambda);
        KCHECK();
        std::swap(xa, ya);
    }
    if (lambda > 0.0 && omega > 1.0 / lambda) return 0.9 / lambda;
    return omega;
}

unsigned long long dbits(double v) {
    unsigned long long b;
    std::memcpy(&b, &v, sizeof b);
    return b;
}

// setup_smoothers (cycle.cpp:32-38): every level, in level order, with the
// reference's error messages. Cached per (kind, omega); null for the kinds
// without setup products (jacobi, gauss_seidel, sor).
const SmSetup* ensure_smoother(gmg_problem* p, int kind, double omega) {
    if (kind == GMG_SMOOTHER_JACOBI || kind == GMG_SMOOTHER_GAUSS_SEIDEL || kind == GMG_SMOOTHER_SOR) return nullptr;
    const auto key = std::make_pair(kind, dbits(omega));
    auto it = p->smsetups.find(key);
    if (it != p->smsetups.end()) return &it->second;
    SmSetup S;
    S.kind = kind;
    S.omega = omega;
    S.lev.resize(p->L);
    try {
        for (int l = 1; l <= p->L; ++l) {
            Lev& L = p->lev(l);
            SmLev& m = S.lev[l - 1];
            if (kind == GMG_SMOOTHER_RICHARDSON) {
                m.rich = richardson_omega(p, L, omega);
            } else if (kind == GMG_SMOOTHER_ILU0) {
                std::vector<double> a[5];
                host_coefs(p, L, a);
                const size_t N = (size_t)L.n();
                std::vector<double> lw(N), ls(N), dp(N);
                gmg_host::factor_ilu0(L.nx, L.ny, a[0].data(), a[1].data(), a[2].data(), a[3].data(), a[4].data(),
                                      lw.data(), ls.data(), dp.data());
                CK(dmalloc(&m.mem, 3 * L.elems * sizeof(double)));
                CK(cudaMemsetAsync(m.mem, 0, 3 * L.elems * sizeof(double), p->st));
                if (g_debug_sync) dbg_sync(__LINE__);
                double* q[3] = {m.mem + L.off0, m.mem + L.elems + L.off0, m.mem + 2 * L.elems + L.off0};
                upload(p, L, q[0], lw.data(), cudaMemcpyHostToDevice);
                upload(p, L, q[1], ls.data(), cudaMemcpyHostToDevice);
                upload(p, L, q[2], dp.data(), cudaMemcpyHostToDevice);
                CK(cudaStreamSynchronize(p->st));
                m.lw = q[0];
                m.ls = q[1];
                m.dp = q[2];
                ensure_scratch(p, L);
            } else {
                const bool fx = uses_x_lines(kind), fy = uses_y_lines(kind);
                const int nset = (int)fx + (int)fy;
                CK(dmalloc(&m.mem, 3 * nset * L.elems * sizeof(double)));
                CK(cudaMemsetAsync(m.mem, 0, 3 * nset * L.elems * sizeof(double), p->st));
                if (g_debug_sync) dbg_sync(__LINE__);
                CK(cudaMemsetAsync(p->status, 0, sizeof(int), p->st));
                if (g_debug_sync) dbg_sync(__LINE__);
                double* base = m.mem + L.off0;
                with_coef(L, [&](const auto& A) {
                    if (fx) {
                        m.fx = LineFactors{base, base + L.elems, base + 2 * L.elems};
                        launch_k(k_tri_factor<0, std::decay_t<decltype(A)>>, (L.ny + 127) / 128, 128, 0, p->st, 
                            L.grid(), A, omega, base, base + L.elems, base + 2 * L.elems, p->status);
                        base += 3 * L.elems;
                    }
                    if (fy) {
                        m.fy = LineFactors{base, base + L.elems, base + 2 * L.elems};
                        launch_k(k_tri_factor<1, std::decay_t<decltype(A)>>, (L.nx + 127) / 128, 128, 0, p->st, 
                            L.grid(), A, omega, base, base + L.elems, base + 2 * L.elems, p->status);
                    }
                });
                KCHECK();
                if (fetch_status(p) == 4) {
                    CK(cudaMemsetAsync(p->status, 0, sizeof(int), p->st));
                    if (g_debug_sync) dbg_sync(__LINE__);
                    throw std::runtime_error("tri factorization: zero pivot");
                }
                if (kind == GMG_SMOOTHER_ADI || kind == GMG_SMOOTHER_GSADI) ensure_scratch(p, L);
            }
        }
    } catch (...) {
        for (auto& m : S.lev) dfree(m.mem);
        throw;
    }
    return &p->smsetups.emplace(key, std::move(S)).first->second;
}

const SmSetup* find_smoother(gmg_problem* p, const gmg_cycle_desc& sp) {
    return ensure_smoother(p, sp.smoother_kind, sp.smoother_omega);
}

// Row slabs: every slab's rows of the finest x to every slab (then slab 0 holds x).
void collect_x(gmg_problem* p, int par) {
    if (!p->dist || p->dist->Ls > p->L) return;
    DistCtx& D = *p->dist;
    dist_gather(driver_slabs(p), D, p->L, par == 0 ? B_X0 : B_X1, D.w0[p->L - 1], D.w1[p->L - 1]);
}

// gmg::solve (cycle.cpp:146-194). b, x in device layout already (B, X[0]).
void solve_core(gmg_problem* p, const gmg_cycle_desc& sp, gmg_solve_report* rep, int* final_par) {
    const auto t0 = std::chrono::steady_clock::now();
    auto elapsed = [&] { return std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count(); };
    check_smoother(sp);
    check_periodic_kind(p, sp.smoother_kind);
    if (p->dist && sp.smoother_kind != GMG_SMOOTHER_JACOBI)
        throw GmgError{GMG_ERR_UNSUPPORTED, "row slabs: only the jacobi smoother is sharded"};
    const SmSetup* sm = ensure_smoother(p, sp.smoother_kind, sp.smoother_omega);
    const int L = p->L;
    const std::vector<gmg_problem*> S = driver_slabs(p);
    for (auto* q : S) CK(cudaMemsetAsync(q->status, 0, sizeof(int), q->st));
    // r0 = ||b - A x||, and the F-cycle's first defect cascade seed
    Driver d0{S, sp, sm};
    d0.initial_resid();
    d0.norm_d(L, DCAS, 2);
    const double r0 = std::sqrt(fetch_scalar(p, p->sums + 2));
    d0.norm_d(L, B_B, 3);
    const double bnorm = std::sqrt(fetch_scalar(p, p->sums + 3));
    int hl = 0;
    rep->residual_history[hl++] = r0;
    rep->iterations = 0;
    rep->converged = 0;
    *final_par = 0;
    const double reference = bnorm > 0.0 ? bnorm : r0;
    if (r0 <= sp.tolerance * reference) {
        rep->converged = 1;
        rep->history_len = hl;
        rep->wall_seconds = elapsed();
        return;
    }
    check_cycle(p, sp);
    // GMG_NO_GRAPH=1 runs the cycle's launches directly (debugging with CUDA_LAUNCH_BLOCKING)
    static const bool no_graph = getenv("GMG_NO_GRAPH") != nullptr;
    auto& ex = no_graph ? p->graphs[""] : get_graphs(p, sp);
    int par = 0;
    for (int k = 1; k <= sp.max_cycles; ++k) {
        if (no_graph) {
            Driver d{driver_slabs(p), sp, find_smoother(p, sp)};
            d.cycle(par == 0 ? B_X0 : B_X1, par == 0 ? B_X1 : B_X0);
            CK(cudaStreamSynchronize(p->st));
        } else {
            CK(cudaGraphLaunch(ex[par], p->st));
        }
        par = 1 - par;
        // ||r||^2 and the adaptive-omega status in one synchronisation (pinned host buffer)
        CK(cudaMemcpyAsync(p->hostbuf, p->sums + 2, sizeof(double), cudaMemcpyDeviceToHost, p->st));
        int* st_host = reinterpret_cast<int*>(p->hostbuf + 1);
        if (sp.adaptive_correction)
            CK(cudaMemcpyAsync(st_host, p->status, sizeof(int), cudaMemcpyDeviceToHost, p->st));
        CK(cudaStreamSynchronize(p->st));
        const double rk = std::sqrt(p->hostbuf[0]);
        if (sp.adaptive_correction && *st_host == 3) {
            rep->history_len = hl;
            throw std::runtime_error("adaptive_omega: correction has nonpositive energy");
        }
        *final_par = par;
        if (rep->convergence_factors) rep->convergence_factors[k - 1] = rk / rep->residual_history[hl - 1];
        rep->residual_history[hl++] = rk;
        rep->iterations = k;
        if (rk <= sp.tolerance * reference) {
            rep->converged = 1;
            break;
        }
        if (rk > 1e6 * std::max(r0, reference)) {
            rep->history_len = hl;
            rep->wall_seconds = elapsed();
            throw GmgError{GMG_DIVERGED, "solve: residual grew beyond 1e6 times the initial residual"};
        }
    }
    rep->history_len = hl;
    rep->wall_seconds = elapsed();
}

void free_problem(gmg_problem* p) {
    if (!p) return;
    cudaSetDevice(p->device);
    if (p->dist && p->dist->local && p->rank == 0) {
        auto D = p->dist;  // keep the context alive while the other slabs go
        for (auto* q : D->slabs)
            if (q != p) free_problem(q);
        D->slabs.clear();
    }
    dfree(p->dscr);
    for (auto& kv : p->graphs)
        for (auto g : kv.second)
            if (g) cudaGraphExecDestroy(g);
    for (auto& kv : p->smsetups)
        for (auto& m : kv.second.lev) dfree(m.mem);
    dfree(p->linebuf);
    for (auto& L : p->lv) {
        dfree(L.scrmem);
        dfree(L.mem);
        dfree(L.coefmem);
        dfree(L.wmem);
    }
    dfree(p->xmem);
    dfree(p->band);
    dfree(p->cscr);
    dfree(p->csum);
    dfree(p->T);
    dfree(p->lb);
    dfree(p->lbs);
    dfree(p->flags);
    dfree(p->recs);
    dfree(p->recs2);
    dfree(p->ss_stats);
    dfree(p->gs_edge);
    dfree(p->gs_state);
    dfree(p->sums);
    dfree(p->nz);
    dfree(p->nz_slots);
    dfree(p->status);
    if (p->hostbuf) cudaFreeHost(p->hostbuf);
    if (p->stage) cudaFreeHost(p->stage);
    for (auto e : p->stage_ev)
        if (e) cudaEventDestroy(e);
    if (p->ev0) cudaEventDestroy(p->ev0);
    if (p->ev1) cudaEventDestroy(p->ev1);
    if (p->st && p->owns_stream) cudaStreamDestroy(p->st);
    delete p;
}

// c (and so RN(1/c)) inside the range where div_rcp is exact (common.cuh)
bool rcp_range_ok(double c) {
    const double a = std::fabs(c);
    return std::isnormal(c) && a >= 0x1p-500 && a <= 0x1p500;
}

double* alloc_pitched(size_t n_buffers, Lev& L) {
    double* m = nullptr;
    CK(dmalloc(&m, n_buffers * L.elems * sizeof(double)));
    return m;
}

void create_problem(const gmg_problem_desc* d, gmg_problem** out) {
    if (!d || d->num_levels < 1 || !d->levels) throw std::logic_error("problem: missing level data");
    std::unique_ptr<gmg_problem, void (*)(gmg_problem*)> p(new gmg_problem, free_problem);
    p->L = d->num_levels;
    p->device = d->device;
    int ndev = 0;
    if (cudaGetDeviceCount(&ndev) != cudaSuccess || ndev == 0)
        throw GmgError{GMG_ERR_CUDA, "no CUDA device available"};
    CK(cudaSetDevice(p->device));
    CK(cudaStreamCreateWithFlags(&p->st, cudaStreamNonBlocking));
    if (!getenv("GMG_NO_PRELOAD")) preload_seqsum_kernels();
    CK(cudaEventCreate(&p->ev0));
    CK(cudaEventCreate(&p->ev1));
    CK(cudaMallocHost(&p->hostbuf, 4 * sizeof(double)));
    p->lv.resize(p->L);
    std::vector<gmg_host::Level> hl(p->L);
    for (int l = 1; l <= p->L; ++l) {
        const gmg_level_desc& ld = d->levels[l - 1];
        if (ld.level != l || ld.nx < 1 || ld.ny < 1) throw std::logic_error("problem: bad level description");
        gmg_host::Level& h = hl[l - 1];
        h.level = l;
        h.nx = ld.nx;
        h.ny = ld.ny;
        h.periodic = d->periodic_y != 0;
        h.x.assign(ld.x, ld.x + ld.nx + 2);
        h.y.assign(ld.y, ld.y + ld.ny + 2);
        if (l >= 2) {
            const std::string err = gmg_host::check_nested(hl[l - 2], h);
            if (!err.empty()) throw std::logic_error("problem: " + err);
        }
        Lev& L = p->lv[l - 1];
        L.l = l;
        L.nx = ld.nx;
        L.ny = ld.ny;
        L.w0 = 0;
        L.w1 = ld.ny;
        // rows 256-B aligned; GMG_PITCH_PAD (multiples of 32 doubles) breaks power-of-two row
        // strides (A/B knob: measured no gain, the HBM address hash already spreads them)
        static const int pitch_pad = [] {
            const char* e = getenv("GMG_PITCH_PAD");
            return e ? (atoi(e) + 31) / 32 * 32 : 0;
        }();
        L.pitch = ((ld.nx + 31) / 32) * 32 + pitch_pad;
        L.off0 = (size_t)L.pitch + 32;
        L.elems = L.off0 + (size_t)(L.ny + 1) * L.pitch + 64;
        L.hx = h.x;
        L.hy = h.y;
        L.mem = alloc_pitched(NBUF, L);
        CK(cudaMemset(L.mem, 0, NBUF * L.elems * sizeof(double)));
        for (int b = 0; b < NBUF; ++b) L.buf[b] = L.mem + b * L.elems + L.off0;
        // operator
        L.per = d->periodic_y != 0;
        const gmg_host::CoefClass cc = gmg_host::classify(ld.nx, ld.ny, ld.c, ld.n, ld.s, ld.e, ld.w, L.per != 0);
        L.kind = cc.kind;
        if (cc.kind == gmg_host::COEF_CONST) {
            L.cconst = CoefConst{cc.c, cc.w, cc.e, cc.s, cc.n, 0.0, 0, 0, 0.0};
            int ex2;
            const double fr = std::frexp(cc.c, &ex2);
            if (fr == 0.5 && std::isnormal(cc.c)) {
                L.cconst.c_pow2 = 1;
                L.cconst.inv_c = std::ldexp(1.0, 1 - ex2);
            }
            if (rcp_range_ok(cc.c)) {
                L.cconst.rcp_ok = 1;
                L.cconst.rcp = 1.0 / cc.c;
            }
        } else if (cc.kind == gmg_host::COEF_ROWX) {
            CK(dmalloc(&L.coefmem, 6 * L.nx * sizeof(double)));
            std::vector<double> rc(L.nx);
            bool ok = true;
            for (int i = 0; i < L.nx; ++i) {
                ok = ok && rcp_range_ok(cc.rc[i]);
                rc[i] = 1.0 / cc.rc[i];
            }
            const std::vector<double>* t[6] = {&cc.rc, &cc.rw, &cc.re, &cc.rs, &cc.rn, &rc};
            for (int q = 0; q < 6; ++q)
                CK(cudaMemcpy(L.coefmem + q * L.nx, t[q]->data(), L.nx * sizeof(double), cudaMemcpyHostToDevice));
            L.crow = CoefRowX{L.coefmem,          L.coefmem + L.nx,     L.coefmem + 2 * L.nx, L.coefmem + 3 * L.nx,
                              L.coefmem + 4 * L.nx, ok ? L.coefmem + 5 * L.nx : nullptr};
        } else if (gmg_host::axis_tables(h, d->coords, d->alpha, d->beta, ld.c, ld.n, ld.s, ld.e, ld.w, L.axt)) {
            // AXES: coefficients on the fly from 1-D tables (checked bit for bit on the host)
            L.kind = 3;
            const gmg_host::AxisTables& T = L.axt;
            const std::vector<double>* tx[7] = {&T.ae, &T.aw, &T.he, &T.hw, &T.mx, &T.rhe, &T.rhw};
            const std::vector<double>* ty[7] = {&T.bn, &T.bs, &T.hn, &T.hs, &T.my, &T.rhn, &T.rhs};
            CK(dmalloc(&L.coefmem, 7 * ((size_t)L.nx + L.ny) * sizeof(double)));
            const double* px[7];
            const double* py[7];
            for (int q = 0; q < 7; ++q) {
                double* dx = L.coefmem + (size_t)q * L.nx;
                double* dy = L.coefmem + 7 * (size_t)L.nx + (size_t)q * L.ny;
                CK(cudaMemcpy(dx, tx[q]->data(), L.nx * sizeof(double), cudaMemcpyHostToDevice));
                CK(cudaMemcpy(dy, ty[q]->data(), L.ny * sizeof(double), cudaMemcpyHostToDevice));
                px[q] = dx;
                py[q] = dy;
            }
            L.caxes = CoefAxes{px[0], px[1], px[2], px[3], px[4], px[5], px[6],
                               py[0], py[1], py[2], py[3], py[4], py[5], py[6], L.nx, L.ny};
        } else {
            CK(dmalloc(&L.coefmem, 5 * L.elems * sizeof(double)));
            CK(cudaMemset(L.coefmem, 0, 5 * L.elems * sizeof(double)));
            const double* src[5] = {ld.c, ld.w, ld.e, ld.s, ld.n};
            double* dst[5];
            for (int q = 0; q < 5; ++q) {
                dst[q] = L.coefmem + q * L.elems + L.off0;
                CK(cudaMemcpy2D(dst[q], L.pitch * sizeof(double), src[q], L.nx * sizeof(double),
                                L.nx * sizeof(double), L.ny, cudaMemcpyHostToDevice));
            }
            L.cfield = CoefField{dst[0], dst[1], dst[2], dst[3], dst[4], L.pitch};
        }

    }
    // transfer tables: tx, ty (fine side); restriction weights (coarse side)
    for (int l = 1; l <= p->L; ++l) {
        Lev& L = p->lv[l - 1];
        std::vector<double> host;
        size_t o_tx = 0, o_ty = 0, o_r = 0;
        if (l >= 2) {
            const Lev& C = p->lv[l - 2];
            auto tx = gmg_host::prolong_weights(L.hx, C.hx, L.nx);
            auto ty = gmg_host::prolong_weights(L.hy, C.hy, L.ny);
            o_tx = host.size();
            host.insert(host.end(), tx.begin(), tx.end());
            o_ty = host.size();
            host.insert(host.end(), ty.begin(), ty.end());
        }
        if (l < p->L) {
            const Lev& Fn = p->lv[l];
            std::vector<double> a, b, c, e, f, g;
            gmg_host::restrict_weights(Fn.hx, L.hx, L.nx, a, b, c);
            gmg_host::restrict_weights(Fn.hy, L.hy, L.ny, e, f, g);
            o_r = host.size();
            for (auto* v : {&a, &b, &c, &e, &f, &g}) host.insert(host.end(), v->begin(), v->end());
        }
        if (host.empty()) continue;
        CK(dmalloc(&L.wmem, host.size() * sizeof(double)));
        CK(cudaMemcpy(L.wmem, host.data(), host.size() * sizeof(double), cudaMemcpyHostToDevice));
        if (l >= 2) {
            L.tx = L.wmem + o_tx;
            L.ty = L.wmem + o_ty;
        }
        if (l < p->L) {
            double* r = L.wmem + o_r;
            L.rw = RestrictW{r, r + L.nx, r + 2 * L.nx, r + 3 * L.nx, r + 3 * L.nx + L.ny,
                             r + 3 * L.nx + 2 * L.ny};
        }
    }
    // level-1 factorization (MultilevelProblem ctor, cycle.cpp:29)
    {
        const gmg_level_desc& ld = d->levels[0];
        const bool per = d->periodic_y != 0;
        std::vector<double> band = per ? gmg_host::cholesky_periodic(ld.c, ld.w, ld.e, ld.s, ld.n, ld.nx, ld.ny)
                                       : gmg_host::cholesky_band(ld.c, ld.w, ld.s, ld.nx, ld.ny);
        p->cn = ld.nx * ld.ny;
        p->cbw = per ? p->cn - 1 : ld.nx;
        CK(dmalloc(&p->band, band.size() * sizeof(double)));
        CK(cudaMemcpy(p->band, band.data(), band.size() * sizeof(double), cudaMemcpyHostToDevice));
        CK(dmalloc(&p->cscr, std::max(1, p->cn) * sizeof(double)));
    }
    // finest x (ping-pong) and b
    {
        Lev& F = p->lv.back();
        CK(dmalloc(&p->xmem, 3 * F.elems * sizeof(double)));
        CK(cudaMemset(p->xmem, 0, 3 * F.elems * sizeof(double)));
        p->X[0] = p->xmem + F.off0;
        p->X[1] = p->xmem + F.elems + F.off0;
        p->B = p->xmem + 2 * F.elems + F.off0;
        const long long n = F.n();
        // chunks of the largest sum: large chunks for the finest level, small chunks up to
        // ss_small_max() terms; >= 2: k_ss_scan2 keeps 2 CTA slots in cincl
        p->nch_max = (int)std::max<long long>(
            {2, (n + kSsC - 1) / kSsC, (std::min<long long>(n, ss_small_max()) + kSsCs - 1) / kSsCs});
        const size_t nm = p->nch_max;
        CK(dmalloc(&p->csum, 2 * nm * sizeof(double)));
        CK(dmalloc(&p->T, 2 * (size_t)n * sizeof(double)));
        CK(dmalloc(&p->lb, 2 * 2 * nm * sizeof(double)));
        CK(cudaMemset(p->lb, 0, 2 * 2 * nm * sizeof(double)));  // look-back words start empty
        CK(dmalloc(&p->lbs, 2 * 2 * nm * sizeof(ChunkAgg)));
        CK(dmalloc(&p->flags, 2 * (2 + 2 * nm) * sizeof(int)));
        CK(cudaMemset(p->flags, 0, 2 * (2 + 2 * nm) * sizeof(int)));
        // records: at most kSsRMax per chunk (a chunk with more stores one literal-resum marker)
        p->rec_cap = (int)std::min<size_t>(nm * kSsRMax, (size_t)INT_MAX / 2);
        CK(dmalloc(&p->recs, 2 * (size_t)p->rec_cap * sizeof(gmg_ss::Rec)));
        CK(dmalloc(&p->recs2, 2 * (size_t)p->rec_cap * sizeof(gmg_ss::Rec)));
        CK(dmalloc(&p->ss_stats, 16 * sizeof(unsigned long long)));
        int maxny = 0, maxnx = 0;
        for (const Lev& Lq : p->lv) {
            maxny = std::max(maxny, Lq.ny);
            maxnx = std::max(maxnx, Lq.nx);
        }
        p->gs_warps = (maxny + 31) / 32;
        p->gs_epitch = (maxnx + 31) / 32 * 32;
        CK(dmalloc(&p->gs_edge, (size_t)p->gs_warps * p->gs_epitch * sizeof(longlong2)));
        CK(cudaMemset(p->gs_edge, 0, (size_t)p->gs_warps * p->gs_epitch * sizeof(longlong2)));
        CK(dmalloc(&p->gs_state, 2 * sizeof(long long)));
        CK(cudaMemset(p->gs_state, 0, 2 * sizeof(long long)));
        CK(dmalloc(&p->linebuf, 2 * (size_t)std::max(maxnx, maxny) * sizeof(double)));
        CK(cudaMemset(p->ss_stats, 0, 16 * sizeof(unsigned long long)));
        CK(dmalloc(&p->sums, 8 * sizeof(double)));
        CK(cudaMemset(p->sums, 0, 8 * sizeof(double)));
        CK(dmalloc(&p->nz, sizeof(int)));
        CK(dmalloc(&p->nz_slots, gmg_problem::kNzSlots * sizeof(int)));
        CK(cudaMemset(p->nz_slots, 0, gmg_problem::kNzSlots * sizeof(int)));
        p->nz_cur = p->nz;
        CK(dmalloc(&p->status, sizeof(int)));
        CK(cudaMemset(p->status, 0, sizeof(int)));
    }
    CK(cudaDeviceSynchronize());
    *out = p.release();
}

DistCtx::~DistCtx() {
    if (!local && comm && nccl().commDestroy) nccl().commDestroy(comm);
}

// Row-slab problem(s): sl->rank < 0 builds all sl->world slabs
// in this process on one device and one stream (virtual ranks; the handle is
// slab 0, which owns the others); sl->rank >= 0 builds this process's slab of
// a multi-process (one GPU per rank) NCCL group.
void create_slabs(const gmg_problem_desc* d, const gmg_slab_desc* sl, gmg_problem** out) {
    if (!sl || sl->world < 1) throw std::invalid_argument("slabs: world must be >= 1");
    if (d && d->periodic_y) throw std::invalid_argument("slabs: periodic (polar) levels are not sharded");
    const bool local = sl->rank < 0;
    if (!local && (sl->rank >= sl->world || !sl->nccl_id)) throw std::invalid_argument("slabs: bad rank or id");
    const int nloc = local ? sl->world : 1;
    std::vector<gmg_problem*> slabs;
    auto D = std::make_shared<DistCtx>();
    try {
        for (int r = 0; r < nloc; ++r) {
            gmg_problem* q = nullptr;
            create_problem(d, &q);
            slabs.push_back(q);
        }
        for (int r = 1; r < nloc; ++r) {
            CK(cudaStreamDestroy(slabs[r]->st));
            slabs[r]->st = slabs[0]->st;
            slabs[r]->owns_stream = false;
        }
        std::vector<int> ny;
        for (int l = 1; l <= d->num_levels; ++l) ny.push_back(d->levels[l - 1].ny);
        const gmg_host::SlabPlan plan = gmg_host::slab_plan(ny, sl->world, std::max(1, sl->min_rows), D->H);
        D->world = sl->world;
        D->Ls = plan.Ls;
        D->local = local;
        D->w0 = plan.w0;
        D->w1 = plan.w1;
        if (!local) {
            NcclId id;
            std::memcpy(id.internal, sl->nccl_id, sizeof id.internal);
            void* comm = nullptr;
            NC(nccl().commInitRank(&comm, sl->world, id, sl->rank));
            D->comm = comm;
        }
        for (int r = 0; r < nloc; ++r) {
            gmg_problem* q = slabs[r];
            q->rank = local ? r : sl->rank;
            q->dist = D;
            for (int l = 1; l <= q->L; ++l) {
                q->lev(l).w0 = plan.w0[l - 1][q->rank];
                q->lev(l).w1 = plan.w1[l - 1][q->rank];
            }
            CK(dmalloc(&q->dscr, (32 + 8 * (size_t)sl->world) * sizeof(double)));
            CK(cudaMemset(q->dscr, 0, (32 + 8 * (size_t)sl->world) * sizeof(double)));
        }
        CK(cudaDeviceSynchronize());
        D->slabs = local ? slabs : std::vector<gmg_problem*>{slabs[0]};
    } catch (...) {
        for (auto* q : slabs) {
            q->dist.reset();
            free_problem(q);
        }
        throw;
    }
    *out = slabs[0];
}

gmg_problem* checked(gmg_problem* p) {
    if (!p) throw std::logic_error("null problem handle");
    CK(cudaSetDevice(p->device));
    return p;
}

void single(const gmg_problem* p, const char* what) {
    if (p->dist) throw std::logic_error(std::string(what) + ": not available on a row-slab handle");
}

void check_level(const gmg_problem* p, int level, const char* what) {
    if (level < 1 || level > p->L) throw std::logic_error(std::string(what) + ": level out of range");
}

}  // namespace

// ============================================================================
// C ABI
// ============================================================================
extern "C" {

const char* gmg_last_error(void) { return g_last_error.c_str(); }

const char* gmg_version(void) { return "gmg_b200 sm_100a; exact-order seqsum v3 (chunk 8192, look-back run carry, tie-parity segments)"; }

int gmg_dev_problem_create(const gmg_problem_desc* desc, gmg_problem** out) {
    return guarded([&] { create_problem(desc, out); });
}

int gmg_dev_problem_destroy(gmg_problem* p) {
    free_problem(p);
    return GMG_OK;
}

int gmg_dev_problem_create_slabs(const gmg_problem_desc* desc, const gmg_slab_desc* slabs, gmg_problem** out) {
    return guarded([&] { create_slabs(desc, slabs, out); });
}

int gmg_dist_unique_id(unsigned char* id128) {
    return guarded([&] {
        NcclId id;
        NC(nccl().getUniqueId(&id));
        std::memcpy(id128, id.internal, sizeof id.internal);
    });
}

int gmg_dev_dist_info(const gmg_problem* p, int* rank, int* world, int* first_sharded_level) {
    return guarded([&] {
        if (!p) throw std::logic_error("null problem handle");
        *rank = p->rank;
        *world = p->dist ? p->dist->world : 1;
        *first_sharded_level = p->dist ? p->dist->Ls : p->L + 1;
    });
}

int gmg_dev_level_window(const gmg_problem* p, int level, int* w0, int* w1) {
    return guarded([&] {
        check_level(p, level, "level_window");
        *w0 = p->lv[level - 1].w0;
        *w1 = p->lv[level - 1].w1;
    });
}

int gmg_dev_num_levels(const gmg_problem* p) { return p ? p->L : 0; }

int gmg_dev_level_shape(const gmg_problem* p, int level, int* nx, int* ny) {
    return guarded([&] {
        check_level(p, level, "level_shape");
        *nx = p->lv[level - 1].nx;
        *ny = p->lv[level - 1].ny;
    });
}

int gmg_dev_level_coef_kind(const gmg_problem* p, int level) {
    if (!p || level < 1 || level > p->L) return -1;
    return p->lv[level - 1].kind;
}

int gmg_dev_solve(gmg_problem* p, const gmg_cycle_desc* spec, const double* b, double* x,
                  gmg_solve_report* rep) {
    return guarded([&] {
        checked(p);
        std::lock_guard<std::mutex> lk(p->mu);
        Lev& F = p->lev(p->L);
        for (auto* q : driver_slabs(p)) {
            upload(q, F, q->B, b, cudaMemcpyHostToDevice);
            upload(q, F, q->X[0], x, cudaMemcpyHostToDevice);
        }
        int par = 0;
        try {
            solve_core(p, *spec, rep, &par);
        } catch (const GmgError& e) {
            if (e.code == GMG_DIVERGED) {
                collect_x(p, par);
                download(p, F, x, p->X[par], cudaMemcpyDeviceToHost);
                CK(cudaStreamSynchronize(p->st));
                std::snprintf(rep->message, sizeof rep->message, "%s", e.msg.c_str());
            }
            throw;
        } catch (const std::runtime_error&) {
            // x keeps the last completed iterate, as the reference's in-place x does
            collect_x(p, par);
            download(p, F, x, p->X[par], cudaMemcpyDeviceToHost);
            CK(cudaStreamSynchronize(p->st));
            throw;
        }
        collect_x(p, par);
        download(p, F, x, p->X[par], cudaMemcpyDeviceToHost);
        CK(cudaStreamSynchronize(p->st));
    });
}

int gmg_dev_solve_devptr(gmg_problem* p, const gmg_cycle_desc* spec, const double* b_dev, double* x_dev,
                         gmg_solve_report* rep) {
    return guarded([&] {
        checked(p);
        std::lock_guard<std::mutex> lk(p->mu);
        Lev& F = p->lev(p->L);
        for (auto* q : driver_slabs(p)) {
            upload(q, F, q->B, b_dev, cudaMemcpyDeviceToDevice);
            upload(q, F, q->X[0], x_dev, cudaMemcpyDeviceToDevice);
        }
        int par = 0;
        solve_core(p, *spec, rep, &par);
        collect_x(p, par);
        download(p, F, x_dev, p->X[par], cudaMemcpyDeviceToDevice);
        CK(cudaStreamSynchronize(p->st));
    });
}

int gmg_dev_mg_cycle(gmg_problem* p, const gmg_cycle_desc* spec, int level, const double* u0,
                     const double* g, double* u) {
    return guarded([&] {
        checked(p);
        single(p, "mg_cycle");
        std::lock_guard<std::mutex> lk(p->mu);
        check_level(p, level, "mg_cycle");
        check_smoother(*spec);
        check_periodic_kind(p, spec->smoother_kind);
        const SmSetup* sm = ensure_smoother(p, spec->smoother_kind, spec->smoother_omega);
        check_cycle(p, *spec);
        Lev& L = p->lev(level);
        // stage u0 in X-side scratch: use DD for g and DCAS for u0 of this level
        upload(p, L, L.buf[DCAS], u0, cudaMemcpyHostToDevice);
        upload(p, L, L.buf[GRHS], g, cudaMemcpyHostToDevice);
        CK(cudaMemsetAsync(p->status, 0, sizeof(int), p->st));
        if (g_debug_sync) dbg_sync(__LINE__);
        Driver d{{p}, *spec, sm};
        SrcId s;
        s.kind = S_U;
        s.u = DCAS;
        // visit() writes level-l results into U0/U1, so g must not alias them: it lives in GRHS,
        // which the recursion only writes on level l-1.
        const int r = d.visit(level, s, GRHS);
        download(p, L, u, L.buf[r], cudaMemcpyDeviceToHost);
        CK(cudaStreamSynchronize(p->st));
        if (spec->adaptive_correction && fetch_status(p) == 3)
            throw std::runtime_error("adaptive_omega: correction has nonpositive energy");
    });
}

int gmg_dev_make_start_vector(gmg_problem* p, const gmg_cycle_desc* spec, int kind, const double* b, double* x) {
    return guarded([&] {
        checked(p);
        single(p, "make_start_vector");
        std::lock_guard<std::mutex> lk(p->mu);
        const int L = p->L;
        Lev& F = p->lev(L);
        if (kind == 0) {  // StartVectorKind::zero
            std::memset(x, 0, (size_t)F.n() * sizeof(double));
            return;
        }
        if (kind != 1) throw std::invalid_argument("start: kind must be zero or nested");
        // nested (study.cpp:46-58): rhs[L] = b, rhs[l-1] = R rhs[l] (the DCAS buffers)
        upload(p, F, F.buf[DCAS], b, cudaMemcpyHostToDevice);
        int cur = U0;
        if (L == 1) {
            launch_coarse(p, F.buf[DCAS], F.buf[U0]);
        } else {
            for (int l = L; l >= 2; --l) launch_restrict(p, l, p->lev(l).buf[DCAS], p->lev(l - 1).buf[DCAS]);
            check_smoother(*spec);
            check_periodic_kind(p, spec->smoother_kind);
            const SmSetup* sm = ensure_smoother(p, spec->smoother_kind, spec->smoother_omega);
            if (!(spec->smoothing_omega > 0.0)) throw std::invalid_argument("omega: damping must be > 0");
            // u = coarse_solver().solve(rhs[1]); per level u = smooth_step(P u, rhs[l])
            launch_coarse(p, p->lev(1).buf[DCAS], p->lev(1).buf[U0]);
            for (int l = 2; l <= L; ++l) {
                Lev& Lv = p->lev(l);
                SmoothSrc s;
                s.kind = S_PROLONG;
                s.uc = p->lev(l - 1).buf[cur];
                if (spec->smoother_kind == GMG_SMOOTHER_JACOBI) {
                    launch_smooth(p, Lv, 1, s, Lv.buf[DCAS], Lv.buf[U0], spec->smoothing_omega);
                    cur = U0;
                } else {
                    const double* r = pc_steps(p, Lv, 1, s, Lv.buf[DCAS], Lv.buf[U0], Lv.buf[U1], *spec,
                                               sm ? &sm->lev[l - 1] : nullptr);
                    cur = r == Lv.buf[U0] ? U0 : U1;
                }
            }
        }
        download(p, F, x, F.buf[cur], cudaMemcpyDeviceToHost);
        CK(cudaStreamSynchronize(p->st));
    });
}

int gmg_dev_apply(gmg_problem* p, int level, const double* x, double* y) {
    return guarded([&] {
        checked(p);
        single(p, "apply");
        std::lock_guard<std::mutex> lk(p->mu);
        check_level(p, level, "apply");
        Lev& L = p->lev(level);
        upload(p, L, L.buf[U0], x, cudaMemcpyHostToDevice);
        with_coef(L, [&](const auto& A) {
            dim3 b(32, 8), gr((L.nx + 31) / 32, (L.ny + 7) / 8);
            launch_k(k_apply_simple<std::decay_t<decltype(A)>>, gr, b, 0, p->st, L.grid(), A, L.buf[U0], L.buf[U1]);
        });
        KCHECK();
        download(p, L, y, L.buf[U1], cudaMemcpyDeviceToHost);
        CK(cudaStreamSynchronize(p->st));
    });
}

int gmg_dev_residual(gmg_problem* p, int level, const double* x, const double* b, double* r) {
    return guarded([&] {
        checked(p);
        single(p, "residual");
        std::lock_guard<std::mutex> lk(p->mu);
        check_level(p, level, "residual");
        Lev& L = p->lev(level);
        upload(p, L, L.buf[U0], x, cudaMemcpyHostToDevice);
        upload(p, L, L.buf[GRHS], b, cudaMemcpyHostToDevice);
        launch_resid(p, L, L.buf[U0], nullptr, L.buf[GRHS], L.buf[DD], nullptr, nullptr);
        download(p, L, r, L.buf[DD], cudaMemcpyDeviceToHost);
        CK(cudaStreamSynchronize(p->st));
    });
}

int gmg_dev_smooth_step(gmg_problem* p, int level, int kind, double somega, double omega_damp,
                        const double* x, const double* b, double* out) {
    return guarded([&] {
        checked(p);
        single(p, "smooth_step");
        std::lock_guard<std::mutex> lk(p->mu);
        check_level(p, level, "smooth_step");
        gmg_cycle_desc sp{};
        sp.smoother_kind = kind;
        sp.smoother_omega = somega;
        check_smoother(sp);
        check_periodic_kind(p, kind);
        const SmSetup* sm = ensure_smoother(p, kind, somega);
        if (!(omega_damp > 0.0)) throw std::invalid_argument("omega: damping must be > 0");
        Lev& L = p->lev(level);
        sp.smoothing_omega = omega_damp;
        upload(p, L, L.buf[U0], x, cudaMemcpyHostToDevice);
        upload(p, L, L.buf[GRHS], b, cudaMemcpyHostToDevice);
        SmoothSrc s;
        s.kind = S_U;
        s.u = L.buf[U0];
        double* r = L.buf[U1];
        if (kind == GMG_SMOOTHER_JACOBI)
            launch_smooth(p, L, 1, s, L.buf[GRHS], L.buf[U1], omega_damp);
        else
            r = pc_steps(p, L, 1, s, L.buf[GRHS], L.buf[U1], L.buf[DCAS], sp, sm ? &sm->lev[level - 1] : nullptr);
        download(p, L, out, r, cudaMemcpyDeviceToHost);
        CK(cudaStreamSynchronize(p->st));
    });
}

int gmg_dev_restriction(gmg_problem* p, int fine_level, const double* fine, double* coarse) {
    return guarded([&] {
        checked(p);
        single(p, "restriction");
        std::lock_guard<std::mutex> lk(p->mu);
        if (fine_level < 2 || fine_level > p->L) throw std::logic_error("restriction: levels are not parent and child");
        Lev& F = p->lev(fine_level);
        Lev& C = p->lev(fine_level - 1);
        upload(p, F, F.buf[U0], fine, cudaMemcpyHostToDevice);
        launch_restrict(p, fine_level, F.buf[U0], C.buf[U1]);
        download(p, C, coarse, C.buf[U1], cudaMemcpyDeviceToHost);
        CK(cudaStreamSynchronize(p->st));
    });
}

int gmg_dev_prolongation(gmg_problem* p, int coarse_level, const double* coarse, double* fine) {
    return guarded([&] {
        checked(p);
        single(p, "prolongation");
        std::lock_guard<std::mutex> lk(p->mu);
        if (coarse_level < 1 || coarse_level >= p->L)
            throw std::logic_error("prolongation: levels are not parent and child");
        Lev& C = p->lev(coarse_level);
        Lev& F = p->lev(coarse_level + 1);
        upload(p, C, C.buf[U0], coarse, cudaMemcpyHostToDevice);
        dim3 b(32, 8), gr((F.nx + 31) / 32, (F.ny + 7) / 8);
        launch_k(k_prolong_simple, gr, b, 0, p->st, prolong_from(p, coarse_level, C.buf[U0]), F.grid(), F.buf[U1]);
        KCHECK();
        download(p, F, fine, F.buf[U1], cudaMemcpyDeviceToHost);
        CK(cudaStreamSynchronize(p->st));
    });
}

int gmg_dev_adaptive_omega(gmg_problem* p, int level, const double* d, const double* corr, double* omega) {
    return guarded([&] {
        checked(p);
        single(p, "adaptive_omega");
        std::lock_guard<std::mutex> lk(p->mu);
        check_level(p, level, "adaptive_omega");
        Lev& L = p->lev(level);
        upload(p, L, L.buf[DD], d, cudaMemcpyHostToDevice);
        upload(p, L, L.buf[U0], corr, cudaMemcpyHostToDevice);
        CK(cudaMemsetAsync(p->nz, 0, sizeof(int), p->st));
        if (g_debug_sync) dbg_sync(__LINE__);
        double* T0 = p->T;
        double* T1 = p->T + p->lev(p->L).n();
        with_coef(L, [&](const auto& A) {
            dim3 b(32, 8), gr((L.nx + 31) / 32, (L.ny + 7) / 8);
            launch_k(k_omega_terms_field<std::decay_t<decltype(A)>>, gr, b, 0, p->st, L.grid(), A, L.buf[DD], L.buf[U0], T0, T1, p->nz);
        });
        KCHECK();
        seqsum(p, ArrTerms{T0, T1}, L.n(), p->sums, GMG_REDUCE_EXACT);
        double h[2];
        int nz = 0;
        CK(cudaMemcpyAsync(h, p->sums, 2 * sizeof(double), cudaMemcpyDeviceToHost, p->st));
        if (g_debug_sync) dbg_sync(__LINE__);
        CK(cudaMemcpyAsync(&nz, p->nz, sizeof(int), cudaMemcpyDeviceToHost, p->st));
        if (g_debug_sync) dbg_sync(__LINE__);
        CK(cudaStreamSynchronize(p->st));
        if (!nz) {
            *omega = 1.0;
            return;
        }
        if (!(h[0] > 0.0)) throw std::runtime_error("adaptive_omega: correction has nonpositive energy");
        *omega = h[1] / h[0];
    });
}

int gmg_dev_coarse_solve(gmg_problem* p, const double* b, double* x) {
    return guarded([&] {
        checked(p);
        single(p, "coarse_solve");
        std::lock_guard<std::mutex> lk(p->mu);
        Lev& L = p->lev(1);
        upload(p, L, L.buf[GRHS], b, cudaMemcpyHostToDevice);
        launch_coarse(p, L.buf[GRHS], L.buf[U0]);
        download(p, L, x, L.buf[U0], cudaMemcpyDeviceToHost);
        CK(cudaStreamSynchronize(p->st));
    });
}

static void flat_sum(gmg_problem* p, long long n, const double* a, const double* b, int mode, double* out) {
    if (n <= 0) {
        *out = 0.0;
        return;
    }
    double *da = nullptr, *db = nullptr;
    CK(dmalloc(&da, n * sizeof(double)));
    if (b) CK(dmalloc(&db, n * sizeof(double)));
    CK(cudaMemcpyAsync(da, a, n * sizeof(double), cudaMemcpyHostToDevice, p->st));
    if (g_debug_sync) dbg_sync(__LINE__);
    if (b) CK(cudaMemcpyAsync(db, b, n * sizeof(double), cudaMemcpyHostToDevice, p->st));
    // a flat vector viewed as one row; chunks never exceed the workspace (checked)
    if ((n + kSsC - 1) / kSsC > p->nch_max) {
        dfree(da);
        dfree(db);
        throw std::logic_error("norm/dot: vector longer than the finest level");
    }
    if (b)
        seqsum(p, DotTerms{da, db}, n, p->sums + 4, mode);
    else
        seqsum(p, FlatNormTerms{da}, n, p->sums + 4, mode);
    *out = fetch_scalar(p, p->sums + 4);
    dfree(da);
    dfree(db);
}

int gmg_dev_norm_l2(gmg_problem* p, long long n, const double* v, int mode, double* out) {
    return guarded([&] {
        checked(p);
        single(p, "norm_l2");
        std::lock_guard<std::mutex> lk(p->mu);
        double s = 0.0;
        flat_sum(p, n, v, nullptr, mode, &s);
        *out = std::sqrt(s);
    });
}

int gmg_dev_dot(gmg_problem* p, long long n, const double* a, const double* b, int mode, double* out) {
    return guarded([&] {
        checked(p);
        single(p, "dot");
        std::lock_guard<std::mutex> lk(p->mu);
        flat_sum(p, n, a, b, mode, out);
    });
}

int gmg_dev_axpy(gmg_problem* p, long long n, double alpha, const double* x, double* y) {
    return guarded([&] {
        checked(p);
        single(p, "axpy");
        std::lock_guard<std::mutex> lk(p->mu);
        if (n <= 0) return;
        double *dx = nullptr, *dy = nullptr;
        CK(dmalloc(&dx, n * sizeof(double)));
        CK(dmalloc(&dy, n * sizeof(double)));
        CK(cudaMemcpyAsync(dx, x, n * sizeof(double), cudaMemcpyHostToDevice, p->st));
        if (g_debug_sync) dbg_sync(__LINE__);
        CK(cudaMemcpyAsync(dy, y, n * sizeof(double), cudaMemcpyHostToDevice, p->st));
        if (g_debug_sync) dbg_sync(__LINE__);
        launch_k(k_axpy_flat, (unsigned)((n + 255) / 256), 256, 0, p->st, n, alpha, dx, dy);
        KCHECK();
        CK(cudaMemcpyAsync(y, dy, n * sizeof(double), cudaMemcpyDeviceToHost, p->st));
        if (g_debug_sync) dbg_sync(__LINE__);
        CK(cudaStreamSynchronize(p->st));
        dfree(dx);
        dfree(dy);
    });
}

int gmg_dev_time_smoother(gmg_problem* p, const gmg_cycle_desc* spec, int variant, int reps, double* ms,
                          double* bytes) {
    return guarded([&] {
        checked(p);
        single(p, "time_smoother");
        std::lock_guard<std::mutex> lk(p->mu);
        if (p->L < 2) throw std::logic_error("time_smoother: needs >= 2 levels");
        const int L = p->L;
        Lev& F = p->lev(L);
        Lev& C = p->lev(L - 1);
        const int M = std::min(std::max(variant == 1 ? spec->post_steps : spec->pre_steps, 1), kMaxFuse);
        SmoothSrc s;
        double per_dof = 24.0;
        if (variant == 0) {
            s.kind = S_PROLONG;
            s.uc = C.buf[U0];
            per_dof = 18.0;
        } else if (variant == 1) {
            s.kind = S_CORRECT;
            s.u = F.buf[U0];
            s.uc = C.buf[U0];
            s.om = OmegaSrc{nullptr, nullptr, 1.0, p->status};
            per_dof = 26.0;
        } else {
            s.kind = S_U;
            s.u = F.buf[U0];
        }
        launch_smooth(p, F, M, s, F.buf[DCAS], F.buf[U1], spec->smoothing_omega);  // warm
        CK(cudaEventRecord(p->ev0, p->st));
        for (int r = 0; r < reps; ++r) launch_smooth(p, F, M, s, F.buf[DCAS], F.buf[U1], spec->smoothing_omega);
        CK(cudaEventRecord(p->ev1, p->st));
        CK(cudaEventSynchronize(p->ev1));
        float t = 0.f;
        CK(cudaEventElapsedTime(&t, p->ev0, p->ev1));
        *ms = (double)t / reps;
        *bytes = per_dof * (double)F.n();
    });
}

int gmg_dev_profile_cycle(gmg_problem* p, const gmg_cycle_desc* spec, const double* b_dev, const double* x_dev,
                          int skip, int cap, gmg_prof_entry* out, int* count) {
    return guarded([&] {
        checked(p);
        std::lock_guard<std::mutex> lk(p->mu);
        check_smoother(*spec);
        const SmSetup* sm = ensure_smoother(p, spec->smoother_kind, spec->smoother_omega);
        check_cycle(p, *spec);
        Lev& F = p->lev(p->L);
        for (auto* q : driver_slabs(p)) {
            upload(q, F, q->B, b_dev, cudaMemcpyDeviceToDevice);
            upload(q, F, q->X[0], x_dev, cudaMemcpyDeviceToDevice);
        }
        // the solve's prologue (r0 and the first defect cascade seed), then `skip` cycles
        Driver d0{driver_slabs(p), *spec, sm};
        d0.initial_resid();
        int par = 0;
        if (skip > 0) {
            auto& ex = get_graphs(p, *spec);
            for (int k = 0; k < skip; ++k, par = 1 - par) CK(cudaGraphLaunch(ex[par], p->st));
        }
        std::vector<ProfEntry> prof;
        prof.reserve(4096);
        struct Reset {
            ~Reset() { g_prof = nullptr; }
        } reset;
        CK(cudaStreamSynchronize(p->st));
        g_prof = &prof;
        try {
            Driver d{driver_slabs(p), *spec, sm};
            d.cycle(par == 0 ? B_X0 : B_X1, par == 0 ? B_X1 : B_X0);
            CK(cudaStreamSynchronize(p->st));
        } catch (...) {
            g_prof = nullptr;
            for (auto& e : prof) {
                cudaEventDestroy(e.e0);
                cudaEventDestroy(e.e1);
            }
            throw;
        }
        g_prof = nullptr;
        int k = 0;
        for (auto& e : prof) {
            float ms = 0.f;
            CK(cudaEventElapsedTime(&ms, e.e0, e.e1));
            if (k < cap) {
                std::snprintf(out[k].kernel, sizeof out[k].kernel, "%s", e.kernel.c_str());
                out[k].level = e.level;
                out[k].bytes = e.bytes;
                out[k].ms = ms;
            }
            ++k;
            cudaEventDestroy(e.e0);
            cudaEventDestroy(e.e1);
        }
        *count = k;
    });
}

int gmg_dev_seqsum_stats(gmg_problem* p, int reset, unsigned long long* out8) {  // 16 values
    return guarded([&] {
        checked(p);
        std::lock_guard<std::mutex> lk(p->mu);
        CK(cudaStreamSynchronize(p->st));
        CK(cudaMemcpy(out8, p->ss_stats, 16 * sizeof(unsigned long long), cudaMemcpyDeviceToHost));
        if (reset) {
            CK(cudaMemsetAsync(p->ss_stats, 0, 16 * sizeof(unsigned long long), p->st));
            if (g_debug_sync) dbg_sync(__LINE__);
            CK(cudaStreamSynchronize(p->st));
        }
    });
}

int gmg_dev_cycle_kernel_count(gmg_problem* p, const gmg_cycle_desc* spec, int* count) {
    return guarded([&] {
        checked(p);
        std::lock_guard<std::mutex> lk(p->mu);
        check_smoother(*spec);
        const SmSetup* sm = ensure_smoother(p, spec->smoother_kind, spec->smoother_omega);
        check_cycle(p, *spec);
        cudaGraph_t g = nullptr;
        CK(cudaStreamBeginCapture(p->st, cudaStreamCaptureModeThreadLocal));
        Driver d{driver_slabs(p), *spec, sm};
        d.cycle(B_X0, B_X1);
        CK(cudaStreamEndCapture(p->st, &g));
        size_t nn = 0;
        CK(cudaGraphGetNodes(g, nullptr, &nn));
        std::vector<cudaGraphNode_t> nodes(nn);
        CK(cudaGraphGetNodes(g, nodes.data(), &nn));
        int k = 0;
        for (auto n : nodes) {
            cudaGraphNodeType t;
            CK(cudaGraphNodeGetType(n, &t));
            if (t == cudaGraphNodeTypeKernel) ++k;
        }
        cudaGraphDestroy(g);
        *count = k;
    });
}

int gmg_host_problem_create(int num_levels, int cnx, int cny, double gx, double gy, int coords, double alpha,
                            double beta, int device, gmg_problem** out) {
    return guarded([&] {
        std::vector<gmg_host::Level> lv = gmg_host::build_problem(num_levels, cnx, cny, gx, gy, coords, alpha, beta);
        std::vector<gmg_level_desc> d(lv.size());
        for (size_t q = 0; q < lv.size(); ++q) {
            d[q] = gmg_level_desc{lv[q].level, lv[q].nx, lv[q].ny, lv[q].x.data(), lv[q].y.data(),
                                  lv[q].c.data(), lv[q].n.data(), lv[q].s.data(), lv[q].e.data(),
                                  lv[q].w.data()};
        }
        gmg_problem_desc pd{num_levels, d.data(), device, coords == GMG_POLAR ? 1 : 0, alpha, beta, coords};
        create_problem(&pd, out);
    });
}

int gmg_host_problem_create_slabs(int num_levels, int cnx, int cny, double gx, double gy, int coords, double alpha,
                                  double beta, int device, const gmg_slab_desc* slabs, gmg_problem** out) {
    return guarded([&] {
        std::vector<gmg_host::Level> lv = gmg_host::build_problem(num_levels, cnx, cny, gx, gy, coords, alpha, beta);
        std::vector<gmg_level_desc> d(lv.size());
        for (size_t q = 0; q < lv.size(); ++q) {
            d[q] = gmg_level_desc{lv[q].level, lv[q].nx, lv[q].ny, lv[q].x.data(), lv[q].y.data(),
                                  lv[q].c.data(), lv[q].n.data(), lv[q].s.data(), lv[q].e.data(),
                                  lv[q].w.data()};
        }
        gmg_problem_desc pd{num_levels, d.data(), device, coords == GMG_POLAR ? 1 : 0, alpha, beta, coords};
        create_slabs(&pd, slabs, out);
    });
}

int gmg_host_slab_plan(int num_levels, const int* ny, int world, int min_rows, int halo, int* first_sharded, int* w0,
                       int* w1) {
    return guarded([&] {
        if (num_levels < 1 || world < 1) throw std::invalid_argument("slab_plan: bad sizes");
        const gmg_host::SlabPlan sp =
            gmg_host::slab_plan(std::vector<int>(ny, ny + num_levels), world, min_rows, halo);
        *first_sharded = sp.Ls;
        for (int l = 0; l < num_levels; ++l)
            for (int r = 0; r < world; ++r) {
                w0[l * world + r] = sp.w0[l][r];
                w1[l * world + r] = sp.w1[l][r];
            }
    });
}

void gmg_host_random_vector(long long n, unsigned seed, double* out) {
    std::mt19937 rng(seed);
    std::uniform_real_distribution<double> dist(-1.0, 1.0);
    for (long long k = 0; k < n; ++k) out[k] = dist(rng);
}

int gmg_host_seqsum_emulate(long long n, const double* terms, int threads, int ept, double* out,
                            long long* stats) {
    return guarded([&] {
        if (threads < 1 || ept < 1) throw std::invalid_argument("seqsum_emulate: bad chunking");
        *out = gmg_host::seqsum_emulate(terms, n, threads, ept, stats);
    });
}

}  // extern "C"
