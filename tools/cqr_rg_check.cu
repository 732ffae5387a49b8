// tools/cqr_rg_check.cu -- the register-grid one-CTA CholeskyQR2 kernels
// (cqr_rg.cuh) against the shared-memory ones (cqr.cuh) on the same inputs:
// max relative difference of every output, and event timings (diagnostic).
#include <cuda_runtime.h>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <vector>
#include "../paper_1804_05138_b200/csrc/cqr_rg.cuh"
using namespace rq;
#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { fprintf(stderr, "%s: %s\n", #x, cudaGetErrorString(e)); exit(1); } } while (0)

static double rel(const std::vector<double> &a, const std::vector<double> &b) {
    double d = 0, m = 0;
    for (size_t i = 0; i < a.size(); ++i) { d = fmax(d, fabs(a[i] - b[i])); m = fmax(m, fabs(a[i])); }
    return m > 0 ? d / m : d;
}

template <int NB>
static void run(int bb) {
    const int bbpad = (bb + 7) / 8 * 8;
    int nb = 8;
    while (nb < bbpad) nb *= 2;
    const size_t B = sizeof(double) * bbpad * bbpad;
    std::vector<double> G(bbpad * bbpad, 0.0), G2(bbpad * bbpad, 0.0), Q(bbpad * bbpad, 0.0);
    srand(bb);
    // G = X^T X for a random 4bb x bb X (SPD, moderate condition)
    std::vector<double> X(4 * bb * bb);
    for (auto &v : X) v = rand() / (double)RAND_MAX - 0.5;
    for (int c = 0; c < bb; ++c)
        for (int r = 0; r < bb; ++r) {
            double s = 0;
            for (int t = 0; t < 4 * bb; ++t) s += X[t + r * 4 * bb] * X[t + c * 4 * bb];
            G[r + c * bbpad] = s;
            G2[r + c * bbpad] = (r == c ? 1.0 : 1e-9 / (1.0 + r + c));
            Q[r + c * bbpad] = (rand() / (double)RAND_MAX - 0.5) * 0.2 + (r == c ? 0.7 : 0.0);
        }
    double *dG, *dG2, *dQ, *dQ2, *dRc[2], *dR[2], *dA[2], *dtau[2], *dus[2], *dui[2], *dli[2], *dvt[2];
    int *st, *be;
    unsigned long long *dbg, *nul = nullptr;
    CK(cudaMalloc(&dbg, 8 * 16));
    double *dQ2c;
    CK(cudaMalloc(&dQ2c, sizeof(double) * bbpad * bbpad));
    CK(cudaMalloc(&dG, B)); CK(cudaMalloc(&dG2, B)); CK(cudaMalloc(&dQ, B)); CK(cudaMalloc(&dQ2, B));
    for (int v = 0; v < 2; ++v) {
        CK(cudaMalloc(&dRc[v], B)); CK(cudaMalloc(&dR[v], B)); CK(cudaMalloc(&dA[v], B)); CK(cudaMalloc(&dtau[v], 8 * bbpad));
        CK(cudaMalloc(&dus[v], B)); CK(cudaMalloc(&dui[v], B)); CK(cudaMalloc(&dli[v], B)); CK(cudaMalloc(&dvt[v], B));
    }
    CK(cudaMalloc(&st, 4)); CK(cudaMalloc(&be, 4));
    CK(cudaMemcpy(dG, G.data(), B, cudaMemcpyHostToDevice));
    CK(cudaMemcpy(dG2, G2.data(), B, cudaMemcpyHostToDevice));
    CK(cudaMemcpy(be, &bb, 4, cudaMemcpyHostToDevice));
    const size_t sm = cqr_smem_bytes(nb), smr = cqr_rg_smem_bytes(NB);
    CK(cudaFuncSetAttribute(cqr_chol_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm));
    CK(cudaFuncSetAttribute(cqr_recon_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm));
    CK(cudaFuncSetAttribute(cqr_chol_rg_kernel<NB>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smr));
    CK(cudaFuncSetAttribute(cqr_recon_rg_kernel<NB>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smr));
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0); cudaEventCreate(&e1);
    float t[2][3] = {{0}};
    unsigned long long hc[3][8];
    int hs[2][3];
    for (int rep = 0; rep < 3; ++rep)
        for (int v = 0; v < 2; ++v) {
            for (int pass = 1; pass <= 2; ++pass) {
                CK(cudaMemcpyToSymbol(g_cqr_dbg, v == 1 ? &dbg : &nul, sizeof(dbg)));
                cudaEventRecord(e0);
                if (v == 0) cqr_chol_kernel<<<1, CQR_THREADS, sm>>>(pass == 1 ? dG : dG2, bb, bbpad, nb, pass, be, st, dRc[v], dR[v], nullptr);
                else cqr_chol_rg_kernel<NB><<<1, RG_THREADS, smr>>>(pass == 1 ? dG : dG2, bb, bbpad, pass, be, st, dRc[v], dR[v], nullptr, 0);
                cudaEventRecord(e1);
                CK(cudaEventSynchronize(e1));
                CK(cudaGetLastError());
                float ms;
                cudaEventElapsedTime(&ms, e0, e1);
                t[v][pass - 1] = ms * 1e3f;
                CK(cudaMemcpy(&hs[v][pass - 1], st, 4, cudaMemcpyDeviceToHost));
                if (v == 1) CK(cudaMemcpy(hc[pass - 1], dbg, 8 * 8, cudaMemcpyDeviceToHost));
            }
            CK(cudaMemcpy(dQ, Q.data(), B, cudaMemcpyHostToDevice));
            CK(cudaMemcpy(dQ2c, Q.data(), B, cudaMemcpyHostToDevice));
            CK(cudaMemset(st, 0, 4));
            cudaEventRecord(e0);
            if (v == 0) cqr_recon_kernel<<<1, CQR_THREADS, sm>>>(dQ, bbpad, bb, bbpad, nb, dRc[v], st, dA[v], bbpad, dtau[v], dus[v], dui[v], dli[v], dvt[v]);
            else cqr_recon_rg_kernel<NB><<<2, RG_THREADS, smr>>>(dQ2c, bbpad, dQ, bbpad, bb, bbpad, dRc[v], st, dA[v], bbpad, dtau[v], dus[v], dui[v], dli[v], dvt[v], nullptr, nullptr);
            cudaEventRecord(e1);
            CK(cudaEventSynchronize(e1));
            CK(cudaGetLastError());
            float ms;
            cudaEventElapsedTime(&ms, e0, e1);
            t[v][2] = ms * 1e3f;
            CK(cudaMemcpy(&hs[v][2], st, 4, cudaMemcpyDeviceToHost));
            if (v == 1) CK(cudaMemcpy(hc[2], dbg, 8 * 8, cudaMemcpyDeviceToHost));
            CK(cudaMemcpyToSymbol(g_cqr_dbg, &nul, sizeof(dbg)));
            if (v == 0) CK(cudaMemcpy(dQ2, dQ, B, cudaMemcpyDeviceToDevice));  // reconstructed V top (old)
        }
    auto get = [&](double *p, size_t n) { std::vector<double> h(n); CK(cudaMemcpy(h.data(), p, n * 8, cudaMemcpyDeviceToHost)); return h; };
    const size_t n2 = (size_t)bbpad * bbpad;
    printf("bb %3d (NB %3d): status old %d %d %d new %d %d %d | us old chol %.1f/%.1f recon %.1f  new chol %.1f/%.1f recon %.1f\n",
           bb, NB, hs[0][0], hs[0][1], hs[0][2], hs[1][0], hs[1][1], hs[1][2], t[0][0], t[0][1], t[0][2], t[1][0], t[1][1], t[1][2]);
    for (int pass = 0; pass < 2; ++pass)
        printf("   new chol %d cycles: load %llu loop %llu checks %llu outputs %llu\n", pass + 1, hc[pass][1] - hc[pass][0],
               hc[pass][2] - hc[pass][1], hc[pass][3] - hc[pass][2], hc[pass][4] - hc[pass][3]);
    printf("   new recon cycles: load %llu LU %llu outputs %llu inverse %llu outputs %llu\n", hc[2][1] - hc[2][0],
           hc[2][2] - hc[2][1], hc[2][3] - hc[2][2], hc[2][4] - hc[2][3], hc[2][5] - hc[2][4]);
    printf("   rel diff: Rc %.2e Rinv %.2e A %.2e tau %.2e us %.2e Uinv %.2e linvt %.2e vt %.2e V %.2e\n",
           rel(get(dRc[0], n2), get(dRc[1], n2)), rel(get(dR[0], n2), get(dR[1], n2)), rel(get(dA[0], n2), get(dA[1], n2)),
           rel(get(dtau[0], bb), get(dtau[1], bb)), rel(get(dus[0], n2), get(dus[1], n2)), rel(get(dui[0], n2), get(dui[1], n2)),
           rel(get(dli[0], n2), get(dli[1], n2)), rel(get(dvt[0], n2), get(dvt[1], n2)), rel(get(dQ2, n2), get(dQ, n2)));
}

int main() {
    run<128>(128);
    run<128>(100);
    run<64>(64);
    run<64>(40);
    run<16>(9);
    return 0;
}
