// tools/cqr_bench.cu -- phase timings (clock64 stamps) of the one-CTA
// CholeskyQR2 kernels at bb = 128 (diagnostic).
#include <cuda_runtime.h>
#include <cstdio>
#include <cstdlib>
#include <vector>
#include "../paper_1804_05138_b200/csrc/cqr.cuh"
using namespace rq;
#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { fprintf(stderr, "%s: %s\n", #x, cudaGetErrorString(e)); return 1; } } while (0)

int main() {
    const int bb = 128, bbpad = 128, nb = 128;
    std::vector<double> G(bbpad * bbpad), G2(bbpad * bbpad), Q(bbpad * bbpad);
    srand(1);
    for (int c = 0; c < bb; ++c)
        for (int r = 0; r < bb; ++r) {
            G[r + c * bbpad] = (r == c ? bb : 0.0) + 1.0 / (1.0 + r + c);
            G2[r + c * bbpad] = (r == c ? 1.0 : 1e-9 / (1.0 + r + c));
            Q[r + c * bbpad] = (rand() / (double)RAND_MAX - 0.5) * 0.2 + (r == c ? 0.7 : 0.0);
        }
    double *dG, *dG2, *dR, *dRc, *dQ, *dA, *dtau, *dus, *dui, *dli, *dvt;
    int *st, *be;
    unsigned long long *dbg;
    const size_t B = 8 * bbpad * bbpad;
    CK(cudaMalloc(&dG, B)); CK(cudaMalloc(&dG2, B)); CK(cudaMalloc(&dR, B)); CK(cudaMalloc(&dRc, B)); CK(cudaMalloc(&dQ, B));
    CK(cudaMalloc(&dA, B)); CK(cudaMalloc(&dtau, 8 * bbpad)); CK(cudaMalloc(&dus, B)); CK(cudaMalloc(&dui, B));
    CK(cudaMalloc(&dli, B)); CK(cudaMalloc(&dvt, B));
    CK(cudaMalloc(&st, 4)); CK(cudaMalloc(&be, 4)); CK(cudaMalloc(&dbg, 8 * 16));
    CK(cudaMemcpy(dG, G.data(), B, cudaMemcpyHostToDevice));
    CK(cudaMemcpy(dG2, G2.data(), B, cudaMemcpyHostToDevice));
    CK(cudaMemcpy(be, &bb, 4, cudaMemcpyHostToDevice));
    CK(cudaMemcpyToSymbol(g_cqr_dbg, &dbg, sizeof(dbg)));
    const size_t sm = cqr_smem_bytes(nb);
    CK(cudaFuncSetAttribute(cqr_chol_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm));
    CK(cudaFuncSetAttribute(cqr_recon_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm));
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0); cudaEventCreate(&e1);
    float ms;
    unsigned long long h[8];
    int hs;
    for (int rep = 0; rep < 3; ++rep) {
        for (int pass = 1; pass <= 2; ++pass) {
            cudaEventRecord(e0);
            cqr_chol_kernel<<<1, CQR_THREADS, sm>>>(pass == 1 ? dG : dG2, bb, bbpad, nb, pass, be, st, dRc, dR, nullptr);
            cudaEventRecord(e1);
            CK(cudaEventSynchronize(e1));
            cudaEventElapsedTime(&ms, e0, e1);
            CK(cudaMemcpy(h, dbg, 8 * 5, cudaMemcpyDeviceToHost));
            CK(cudaMemcpy(&hs, st, 4, cudaMemcpyDeviceToHost));
            printf("chol pass %d: %.1f us (status %d); cycles: load %llu, factor %llu, checks+R+Rc %llu, inverse %llu\n", pass,
                   ms * 1e3, hs, h[1] - h[0], h[2] - h[1], h[3] - h[2], h[4] - h[3]);
        }
        CK(cudaMemcpy(dQ, Q.data(), B, cudaMemcpyHostToDevice));
        CK(cudaMemset(st, 0, 4));
        cudaEventRecord(e0);
        cqr_recon_kernel<<<1, CQR_THREADS, sm>>>(dQ, bbpad, bb, bbpad, nb, dRc, st, dA, bbpad, dtau, dus, dui, dli, dvt);
        cudaEventRecord(e1);
        CK(cudaEventSynchronize(e1));
        cudaEventElapsedTime(&ms, e0, e1);
        CK(cudaMemcpy(h, dbg, 8 * 3, cudaMemcpyDeviceToHost));
        CK(cudaMemcpy(&hs, st, 4, cudaMemcpyDeviceToHost));
        printf("recon: %.1f us (status %d); cycles: load+LU %llu, outputs+inverses %llu\n", ms * 1e3, hs, h[1] - h[0], h[2] - h[1]);
    }
    return 0;
}
