// Microbenchmark: dependent-latency of the exact-sum chain's serial step on sm_100a.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o chain_lat chain_lat.cu && ./chain_lat
#include <cstdio>
#include <cstdint>
__global__ void k_dadd(double* out, long long* cyc, double a, int n) {
    double x = a;
    long long t0 = clock64();
    for (int i = 0; i < n; ++i) x = x + a;
    long long t1 = clock64();
    out[0] = x; cyc[0] = t1 - t0;
}
__global__ void k_iadd_dadd(double* out, long long* cyc, double a, long long d, int n) {
    double x = a;
    long long t0 = clock64();
    for (int i = 0; i < n; ++i) x = __longlong_as_double(__double_as_longlong(x) + d) + a;
    long long t1 = clock64();
    out[0] = x; cyc[0] = t1 - t0;
}
// the chain's group loop: 32 records staged in shared memory, lane k's record applied serially
__global__ void k_group(double* out, long long* cyc, int groups) {
    __shared__ longlong2 cD[32];
    __shared__ double2 cPB[32];
    const int lane = threadIdx.x;
    double sv = 1.5;
    long long t0 = clock64();
    for (int g = 0; g < groups; ++g) {
        cD[lane] = make_longlong2(lane & 1, 0);
        cPB[lane] = make_double2(-0.0, 0.0);
        __syncwarp();
        double x = sv, before = sv;
#pragma unroll 8
        for (int k = 0; k < 32; ++k) {
            if (lane == k) before = x;
            x = __longlong_as_double(__double_as_longlong(x) + cD[k].x) + cPB[k].x;
        }
        sv = x + before * 0.0;
        __syncwarp();
    }
    long long t1 = clock64();
    if (lane == 0) { out[0] = sv; cyc[0] = t1 - t0; }
}
// same, operands preloaded into registers by shuffles (no shared memory in the serial loop)
__global__ void k_group_shfl(double* out, long long* cyc, int groups) {
    const int lane = threadIdx.x;
    double sv = 1.5;
    long long t0 = clock64();
    for (int g = 0; g < groups; ++g) {
        const long long dmine = lane & 1;
        const double pmine = -0.0;
        double x = sv, before = sv;
#pragma unroll
        for (int k = 0; k < 32; ++k) {
            const long long dk = __shfl_sync(0xffffffffu, dmine, k);
            const double pk = __shfl_sync(0xffffffffu, pmine, k);
            if (lane == k) before = x;
            x = __longlong_as_double(__double_as_longlong(x) + dk) + pk;
        }
        sv = x + before * 0.0;
    }
    long long t1 = clock64();
    if (lane == 0) { out[0] = sv; cyc[0] = t1 - t0; }
}
// fp64 chain: x = (x + a_k) + p_k, operands broadcast by shuffles
__global__ void k_group_dd(double* out, long long* cyc, int groups) {
    const int lane = threadIdx.x;
    double sv = 1.5, bsum = 0.0;
    long long t0 = clock64();
    for (int g = 0; g < groups; ++g) {
        const double av = (lane & 1) ? 0x1p-52 : -0.0;
        const double pv = -0.0;
        double x = sv, before = sv;
#pragma unroll
        for (int k = 0; k < 32; ++k) {
            const double ak = __shfl_sync(0xffffffffu, av, k);
            const double pk = __shfl_sync(0xffffffffu, pv, k);
            if (lane == k) before = x;
            x = (x + ak) + pk;
        }
        sv = x;
        bsum += before;
    }
    long long t1 = clock64();
    if (lane == 0) { out[0] = sv + bsum; cyc[0] = t1 - t0; }
}
// same with operands from shared memory (written per group)
__global__ void k_group_dd_smem(double* out, long long* cyc, int groups) {
    __shared__ double sa[32], sp[32];
    const int lane = threadIdx.x;
    double sv = 1.5, bsum = 0.0;
    long long t0 = clock64();
    for (int g = 0; g < groups; ++g) {
        sa[lane] = (lane & 1) ? 0x1p-52 : -0.0;
        sp[lane] = -0.0;
        __syncwarp();
        double x = sv, before = sv;
#pragma unroll
        for (int k = 0; k < 32; ++k) {
            if (lane == k) before = x;
            x = (x + sa[k]) + sp[k];
        }
        __syncwarp();
        sv = x;
        bsum += before;
    }
    long long t1 = clock64();
    if (lane == 0) { out[0] = sv + bsum; cyc[0] = t1 - t0; }
}
// tie path, fp64: x = (x + (parity(x) ? a1 : a0)) + p
__global__ void k_group_tie_fp(double* out, long long* cyc, int groups) {
    const int lane = threadIdx.x;
    double sv = 1.5, bsum = 0.0;
    long long t0 = clock64();
    for (int g = 0; g < groups; ++g) {
        const double a0v = (lane & 1) ? 0x1p-52 : -0.0;
        const double a1v = (lane & 2) ? 0x1p-51 : -0.0;
        const double pv = -0.0;
        double x = sv, before = sv;
#pragma unroll
        for (int k = 0; k < 32; ++k) {
            const double a0 = __shfl_sync(0xffffffffu, a0v, k);
            const double a1 = __shfl_sync(0xffffffffu, a1v, k);
            const double pk = __shfl_sync(0xffffffffu, pv, k);
            if (lane == k) before = x;
            const double a = (__double2loint(x) & 1) ? a1 : a0;
            x = (x + a) + pk;
        }
        sv = x;
        bsum += before;
    }
    long long t1 = clock64();
    if (lane == 0) { out[0] = sv + bsum; cyc[0] = t1 - t0; }
}
// tie path: both parity outcomes computed in parallel, selected after
__global__ void k_group_tie_fp2(double* out, long long* cyc, int groups) {
    const int lane = threadIdx.x;
    double sv = 1.5, bsum = 0.0;
    long long t0 = clock64();
    for (int g = 0; g < groups; ++g) {
        const double a0v = (lane & 1) ? 0x1p-52 : -0.0;
        const double a1v = (lane & 2) ? 0x1p-51 : -0.0;
        const double pv = -0.0;
        double x = sv, before = sv;
#pragma unroll
        for (int k = 0; k < 32; ++k) {
            const double a0 = __shfl_sync(0xffffffffu, a0v, k);
            const double a1 = __shfl_sync(0xffffffffu, a1v, k);
            const double pk = __shfl_sync(0xffffffffu, pv, k);
            if (lane == k) before = x;
            const bool odd = __double2loint(x) & 1;
            const double y0 = (x + a0) + pk;
            const double y1 = (x + a1) + pk;
            x = odd ? y1 : y0;
        }
        sv = x;
        bsum += before;
    }
    long long t1 = clock64();
    if (lane == 0) { out[0] = sv + bsum; cyc[0] = t1 - t0; }
}
// mixed: a per-record warp-uniform choice between the plain and the parity step
__global__ void k_group_mixed(double* out, long long* cyc, int groups, unsigned tmask_in) {
    const int lane = threadIdx.x;
    double sv = 1.5, bsum = 0.0;
    long long t0 = clock64();
    for (int g = 0; g < groups; ++g) {
        const unsigned tmask = __shfl_sync(0xffffffffu, tmask_in ^ (unsigned)g * 0, 0);
        const double a0v = (lane & 1) ? 0x1p-52 : -0.0;
        const double a1v = (lane & 2) ? 0x1p-51 : -0.0;
        const double pv = -0.0;
        double x = sv, before = sv;
#pragma unroll
        for (int k = 0; k < 32; ++k) {
            const double a0 = __shfl_sync(0xffffffffu, a0v, k);
            const double pk = __shfl_sync(0xffffffffu, pv, k);
            if (lane == k) before = x;
            if (tmask & (1u << k)) {
                const double a1 = __shfl_sync(0xffffffffu, a1v, k);
                const double a = (__double2loint(x) & 1) ? a1 : a0;
                x = (x + a) + pk;
            } else {
                x = (x + a0) + pk;
            }
        }
        sv = x;
        bsum += before;
    }
    long long t1 = clock64();
    if (lane == 0) { out[0] = sv + bsum; cyc[0] = t1 - t0; }
}
int main() {
    double* o; long long* c; cudaMalloc(&o, 8); cudaMalloc(&c, 8); long long h;
    const int n = 100000;
    k_dadd<<<1, 1>>>(o, c, 1e-300, n); cudaMemcpy(&h, c, 8, cudaMemcpyDeviceToHost);
    printf("dependent DADD: %.2f cycles\n", (double)h / n);
    k_iadd_dadd<<<1, 1>>>(o, c, 1e-300, 1, n); cudaMemcpy(&h, c, 8, cudaMemcpyDeviceToHost);
    printf("dependent IADD64 + DADD: %.2f cycles\n", (double)h / n);
    k_group<<<1, 32>>>(o, c, 2000); cudaMemcpy(&h, c, 8, cudaMemcpyDeviceToHost);
    printf("group loop (smem operands): %.2f cycles/record\n", (double)h / (2000 * 32));
    k_group_shfl<<<1, 32>>>(o, c, 2000); cudaMemcpy(&h, c, 8, cudaMemcpyDeviceToHost);
    printf("group loop (shfl operands): %.2f cycles/record\n", (double)h / (2000 * 32));
    k_group_dd<<<1, 32>>>(o, c, 2000); cudaMemcpy(&h, c, 8, cudaMemcpyDeviceToHost);
    printf("fp64 chain (shfl operands): %.2f cycles/record\n", (double)h / (2000 * 32));
    k_group_dd_smem<<<1, 32>>>(o, c, 2000); cudaMemcpy(&h, c, 8, cudaMemcpyDeviceToHost);
    printf("fp64 chain (smem operands): %.2f cycles/record\n", (double)h / (2000 * 32));
    k_group_tie_fp<<<1, 32>>>(o, c, 2000); cudaMemcpy(&h, c, 8, cudaMemcpyDeviceToHost);
    printf("tie chain fp64 select (shfl operands): %.2f cycles/record\n", (double)h / (2000 * 32));
    k_group_tie_fp2<<<1, 32>>>(o, c, 2000); cudaMemcpy(&h, c, 8, cudaMemcpyDeviceToHost);
    printf("tie chain fp64 both outcomes (shfl operands): %.2f cycles/record\n", (double)h / (2000 * 32));
    for (unsigned m : {0u, 0x00100401u, 0x11111111u, 0xffffffffu}) {
        k_group_mixed<<<1, 32>>>(o, c, 2000, m); cudaMemcpy(&h, c, 8, cudaMemcpyDeviceToHost);
        printf("mixed tie mask %08x: %.2f cycles/record\n", m, (double)h / (2000 * 32));
    }
    return 0;
}
