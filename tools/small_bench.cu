// tools/small_bench.cu -- latency of the small one-CTA building blocks
// (diagnostic): __syncthreads loops, FP64 division, the CholeskyQR2 Cholesky
// kernel, and back-to-back launch overhead.
#include <cuda_runtime.h>
#include <cstdio>
#include <vector>
#include "../paper_1804_05138_b200/csrc/cqr.cuh"
using namespace rq;
#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { fprintf(stderr, "%s: %s\n", #x, cudaGetErrorString(e)); return 1; } } while (0)

__global__ void sync_loop(long long *out, int n, int work) {
    long long t0 = clock64();
    double x = threadIdx.x;
    for (int i = 0; i < n; ++i) {
        for (int w = 0; w < work; ++w) x = x * 0.999 + 1.0 / (x + 3.0);
        __syncthreads();
    }
    long long t1 = clock64();
    if (threadIdx.x == 0) out[0] = t1 - t0;
    if (x == 1234.5) out[1] = 1;
}
__global__ void empty_kernel() {}
__device__ __forceinline__ unsigned long long gtimer() {
    unsigned long long t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    return t;
}
// effective SM clock: cycles / ns over a ~100 us dependent DFMA chain
__global__ void clock_probe(long long *out, int iters) {
    const unsigned long long g0 = gtimer();
    const long long c0 = clock64();
    double x = threadIdx.x;
    for (int i = 0; i < iters; ++i) x = fma(x, 0.999999, 1e-3);
    const long long c1 = clock64();
    const unsigned long long g1 = gtimer();
    if (threadIdx.x == 0) { out[0] = c1 - c0; out[1] = (long long)(g1 - g0); }
    if (x == 1234.5) out[2] = 1;
}

int main() {
    long long *d, h[3];
    CK(cudaMalloc(&d, 32));
    for (int rep = 0; rep < 3; ++rep)
        for (int iters : {1000, 20000, 200000}) {
            clock_probe<<<1, 32>>>(d, iters);
            CK(cudaMemcpy(h, d, 16, cudaMemcpyDeviceToHost));
            printf("clock_probe iters=%d: %lld cycles in %lld ns -> %.0f MHz\n", iters, h[0], h[1], 1e3 * h[0] / (double)h[1]);
        }
    for (int work : {0, 1}) {
        sync_loop<<<1, 256>>>(d, 64, work);
        CK(cudaDeviceSynchronize());
        sync_loop<<<1, 256>>>(d, 64, work);
        CK(cudaMemcpy(h, d, 16, cudaMemcpyDeviceToHost));
        printf("sync_loop work=%d: %lld cycles for 64 steps (%.0f per step)\n", work, h[0], h[0] / 64.0);
    }
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0); cudaEventCreate(&e1);
    for (int i = 0; i < 10; ++i) empty_kernel<<<1, 32>>>();
    cudaEventRecord(e0);
    for (int i = 0; i < 1000; ++i) empty_kernel<<<1, 32>>>();
    cudaEventRecord(e1);
    CK(cudaEventSynchronize(e1));
    float ms; cudaEventElapsedTime(&ms, e0, e1);
    printf("empty kernel back-to-back: %.2f us per launch\n", ms);
    // Cholesky of a 64x64 SPD matrix, with phase stamps
    {
        const int bb = 64, bbpad = 64, nb = 64;
        std::vector<double> G(bbpad * bbpad);
        for (int c = 0; c < bb; ++c)
            for (int r = 0; r < bb; ++r) G[r + c * bbpad] = (r == c ? bb : 0.0) + 1.0 / (1.0 + r + c);
        double *dG, *dR, *dRc;
        int *st, *be;
        unsigned long long *dbg;
        CK(cudaMalloc(&dG, 8 * bbpad * bbpad)); CK(cudaMalloc(&dR, 8 * bbpad * bbpad)); CK(cudaMalloc(&dRc, 8 * bbpad * bbpad));
        CK(cudaMalloc(&st, 4)); CK(cudaMalloc(&be, 4)); CK(cudaMalloc(&dbg, 8 * 16));
        CK(cudaMemcpy(dG, G.data(), 8 * bbpad * bbpad, cudaMemcpyHostToDevice));
        CK(cudaMemcpy(be, &bb, 4, cudaMemcpyHostToDevice));
        CK(cudaMemcpyToSymbol(g_cqr_dbg, &dbg, sizeof(dbg)));
        const size_t sm = ((size_t)nb * nb + (nb / 2) * (nb / 2)) * 8;
        CK(cudaFuncSetAttribute(cqr_chol_kernel<9>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm));
        for (int rep = 0; rep < 3; ++rep) {
            cudaEventRecord(e0);
            cqr_chol_kernel<9><<<1, CQR_THREADS, sm>>>(dG, bb, bbpad, nb, 1, be, st, dRc, dR);
            cudaEventRecord(e1);
            CK(cudaEventSynchronize(e1));
            cudaEventElapsedTime(&ms, e0, e1);
            unsigned long long h[8];
            CK(cudaMemcpy(h, dbg, 8 * 5, cudaMemcpyDeviceToHost));
            int hs; CK(cudaMemcpy(&hs, st, 4, cudaMemcpyDeviceToHost));
            printf("cqr_chol<9> bb=64: %.2f us (status %d); cycles: load %llu, factor %llu, Rc %llu, inverse %llu\n", ms * 1e3, hs,
                   h[1] - h[0], h[2] - h[1], h[3] - h[2], h[4] - h[3]);
        }
    }
    return 0;
}
