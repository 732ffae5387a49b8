// misc.cuh -- S3 swap (K5), S6 sample update (K8), and the sample's
// Frobenius norm for the rank-stop threshold (reading R-G12).
#pragma once
#include "common.cuh"

namespace rq {

// ---------------------------------------------------------------------------
// ||B||_F^2 of the initial sample, deterministic two-level sum; sets
// stop_tol2 = (1e3 eps)^2 ||B||_F^2 and status = 4 if non-finite.
// ---------------------------------------------------------------------------
__global__ void sumsq_partial_kernel(const double *B, int64_t rows, int64_t cols, int64_t ldb, double *part) {
    __shared__ double red[32];
    const int64_t total = rows * cols;
    double s = 0.0;
    for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < total; e += (int64_t)gridDim.x * blockDim.x) {
        const int64_t r = e % rows, c = e / rows;
        const double v = B[r + c * ldb];
        s += v * v;
    }
    s = warp_sum(s);
    if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = s;
    __syncthreads();
    if (threadIdx.x < 32) {
        double t = (threadIdx.x < (blockDim.x >> 5)) ? red[threadIdx.x] : 0.0;
        t = warp_sum(t);
        if (threadIdx.x == 0) part[blockIdx.x] = t;
    }
}

__global__ void sumsq_final_kernel(const double *part, int nparts, double *stop_tol2, int *status) {
    // one warp: lane-strided partial sums, then the fixed butterfly (deterministic)
    double s = 0.0;
    for (int q = threadIdx.x; q < nparts; q += 32) s += part[q];
    s = warp_sum(s);
    if (threadIdx.x != 0) return;
    const double eps = 0x1p-52;
    *stop_tol2 = (1e3 * eps) * (1e3 * eps) * s;
    if (!isfinite(s)) *status = 4;
}

// ---------------------------------------------------------------------------
// S3 swap ("Swap (j1..jb) and (i:i+b-1) columns in A, Pi"): the
// sample QRCP kernel turns its bb_eff transpositions (applied in order,
// reading R-G5) into a list of (dst, src) column moves over the <= 2 bb
// positions they touch.  Whole columns move (full height m, so earlier R12
// rows move with them: LAPACK semantics), through a staging buffer, and
// jpvt with them.
// ---------------------------------------------------------------------------
__global__ void swap_gather_kernel(const double *A /* + i*lda */, int64_t lda, int64_t m, const int64_t *jpvt,
                                   const int64_t *src, const int *npairs, double *stage, int64_t lds,
                                   int64_t *jstage) {
    const int np = *npairs;
    const int64_t total = (int64_t)np * m;
    for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < total; e += (int64_t)gridDim.x * blockDim.x) {
        const int64_t r = e % m, q = e / m;
        stage[r + q * lds] = A[r + src[q] * lda];
        if (r == 0) jstage[q] = jpvt[src[q]];
    }
}

// One-kernel form: CTA b moves rows [b R, b R + R) of every (src -> dst) pair
// through shared memory -- all reads of its rows, then all writes -- so no
// staging buffer and no second launch (rows are independent); CTA 0 also moves
// jpvt.  np <= SW_MAXP pairs.
constexpr int SW_ROWS = 16, SW_MAXP = 256;
__global__ void __launch_bounds__(256) swap_fused_kernel(double *A /* + i*lda */, int64_t lda, int64_t m,
                                                         int64_t *jpvt, const int64_t *src, const int64_t *dst,
                                                         const int *npairs) {
    __shared__ double st[SW_MAXP][SW_ROWS + 1];
    __shared__ int64_t js[SW_MAXP];
    __shared__ int64_t ss[SW_MAXP], ds[SW_MAXP];
    const int np = *npairs;
    const int64_t r0 = (int64_t)blockIdx.x * SW_ROWS;
    for (int q = threadIdx.x; q < np; q += blockDim.x) { ss[q] = src[q]; ds[q] = dst[q]; }
    __syncthreads();
    for (int e = threadIdx.x; e < np * SW_ROWS; e += blockDim.x) {
        const int r = e % SW_ROWS, q = e / SW_ROWS;
        if (r0 + r < m) st[q][r] = A[r0 + r + ss[q] * lda];
    }
    if (blockIdx.x == 0)
        for (int q = threadIdx.x; q < np; q += blockDim.x) js[q] = jpvt[ss[q]];
    __syncthreads();
    for (int e = threadIdx.x; e < np * SW_ROWS; e += blockDim.x) {
        const int r = e % SW_ROWS, q = e / SW_ROWS;
        if (r0 + r < m) A[r0 + r + ds[q] * lda] = st[q][r];
    }
    if (blockIdx.x == 0)
        for (int q = threadIdx.x; q < np; q += blockDim.x) jpvt[ds[q]] = js[q];
}

__global__ void swap_scatter_kernel(double *A, int64_t lda, int64_t m, int64_t *jpvt, const int64_t *dst,
                                    const int *npairs, const double *stage, int64_t lds, const int64_t *jstage) {
    const int np = *npairs;
    const int64_t total = (int64_t)np * m;
    for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < total; e += (int64_t)gridDim.x * blockDim.x) {
        const int64_t r = e % m, q = e / m;
        A[r + dst[q] * lda] = stage[r + q * lds];
        if (r == 0) jpvt[dst[q]] = jstage[q];
    }
}

// ---------------------------------------------------------------------------
// S6 sample update, Eq. (4) (readings R-G1..G3, R-G20):
//   Omega-hat11 = R-hat11 R11^{-1}   (b x b upper triangular; tri.cuh)
//   B_next(0:bb, c) = R-hat12(:, c) - Omega-hat11 R12(:, c)
//   B_next(bb:l, c) = R-hat22(:, c);  rows l..lpad-1 = 0
// R-hat12/22 are read from the physical sample columns through the position
// map perm written by the sample QRCP.  C = Omega-hat11 R12 (bbpad x n'') comes
// from a DMMA contraction; this kernel forms
// B_next(r, c) = R-hat12(r, src) - C(r, c) for r < bb, copies the R-hat22 rows
// and zeroes rows l..lpad-1.  Local output column c = this rank's trailing
// column lj0 + c (global column j = dist_global(lj0 + c), position j - i in the
// replicated sample); P = 1: j = lj0 + c with lj0 = i + bb.
// ---------------------------------------------------------------------------
__global__ void sample_update4_kernel(const double *Bold, int64_t ldb, const int64_t *perm, const double *Cm,
                                      int64_t ldc, int bb, int l, int lpad, int64_t npl, const int *bb_eff,
                                      double *Bnew, int64_t ldn, int64_t i, int64_t lj0, int b, int P, int rank) {
    if (*bb_eff != bb) return;
    const int64_t total = (int64_t)lpad * npl;
    for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < total; e += (int64_t)gridDim.x * blockDim.x) {
        const int r = (int)(e % lpad);
        const int64_t c = e / lpad;
        const int64_t lj = lj0 + c;
        const int64_t j = ((lj / b) * P + rank) * b + lj % b;  // global column (dist_global)
        const int64_t src = perm[j - i];
        double v = 0.0;
        if (r < bb) v = Bold[r + src * ldb] - Cm[r + c * ldc];
        else if (r < l) v = Bold[r + src * ldb];
        Bnew[r + c * ldn] = v;
    }
}

// ---------------------------------------------------------------------------
// S6 by updating formula 2, Eq. (5): B_next = B2 - Omega-bar_1 R12
// with B2 the pre-QRCP sample's columns in pivoted order (perm[bb + ...]) and
// C = Omega-bar_1 R12 (l x n'') computed by a DMMA contraction; this kernel
// forms B2 - C for this rank's local trailing columns (same mapping as
// sample_update4_kernel).  Rows l..lpad-1 are 0.
// ---------------------------------------------------------------------------
__global__ void sample_update5_kernel(const double *Bpre, int64_t ldb, const int64_t *perm, const double *Cm,
                                      int64_t ldc, int bb, int l, int lpad, int64_t npl, const int *bb_eff,
                                      double *Bnew, int64_t ldn, int64_t i, int64_t lj0, int b, int P, int rank) {
    if (*bb_eff != bb) return;
    const int64_t total = (int64_t)lpad * npl;
    for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < total; e += (int64_t)gridDim.x * blockDim.x) {
        const int r = (int)(e % lpad);
        const int64_t c = e / lpad;
        const int64_t lj = lj0 + c;
        const int64_t j = ((lj / b) * P + rank) * b + lj % b;  // global column (dist_global)
        const int64_t src = perm[j - i];
        Bnew[r + c * ldn] = (r < l) ? Bpre[r + src * ldb] - Cm[r + c * ldc] : 0.0;
    }
}

}  // namespace rq
