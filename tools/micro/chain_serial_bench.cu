// Microbenchmark of chain_serial (seqsum.cuh) on synthetic operands: cycles per record for
// groups without ties, with a few ties, and all ties.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -fmad=false --expt-relaxed-constexpr \
//        -I paper_0805_3041_b200/csrc -o chain_serial_bench tools/micro/chain_serial_bench.cu
#include <cstdio>
#include "seqsum.cuh"
using namespace gmg_dev;
__global__ void __launch_bounds__(256) k(double* out, long long* cyc, int tie_every, int reps) {
    extern __shared__ __align__(16) unsigned char raw[];
    ChainSmem& M = *reinterpret_cast<ChainSmem*>(raw);
    const int t = threadIdx.x;
    for (int q = t; q < kSsBatch; q += blockDim.x) {
        M.op[0].d[q] = q & 3;
        M.op[0].ft[q] = (tie_every && q % tie_every == 0) ? 2 | (q & 1) : 0;
        M.op[0].pb[q] = (q & 1) ? -0.0 : 0x1p-60;
    }
    __syncthreads();
    if (t < 32) {
        double sv = 1.5;
        const long long c0 = clock64();
        for (int r = 0; r < reps; ++r) sv = chain_serial(M.op[0], M.before, 0, kSsBatch, sv);
        const long long c1 = clock64();
        if (t == 0) { out[0] = sv; cyc[0] = c1 - c0; }
    }
}
int main() {
    double* o; long long* c; cudaMalloc(&o, 8); cudaMalloc(&c, 8); long long h;
    cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sizeof(ChainSmem));
    for (int te : {0, 32, 7, 1}) {
        k<<<1, 256, sizeof(ChainSmem)>>>(o, c, te, 20);
        cudaError_t e = cudaMemcpy(&h, c, 8, cudaMemcpyDeviceToHost);
        printf("tie every %d: %.2f cycles/record (%s)\n", te, (double)h / (20.0 * kSsBatch), cudaGetErrorString(e));
    }
    return 0;
}
