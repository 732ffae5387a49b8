// srqr.cuh -- SRQR verification (Alg. 3 first half; SURVEY.md
// §8(f) N1) on top of the RQRCP factorization to rank k (the paper's l):
//   1. r_i = ||B(:, i)||^2 / (b + p) over the sample after the last panel's
//      update (kept for this purpose, reading G9), iota = argmax (lowest
//      position on ties, reading G5)                      (srqr_pick_kernel)
//   2. columns k and k + iota of A and Pi swapped (the swap kernels of S3)
//   3. |alpha| = ||A(k:m, k)|| (one QR step) and g1 =
//      ||A(k:m, k:n)||_{1,2} / |alpha| (Eq. 8)           (srqr_norms_kernel)
//   4. Y = R-hat^{-1} Omega_d^T, R-hat = [[R11, a], [0, |alpha|]], Omega_d the
//      d x (k+1) Gaussian of (seed, stream 7): one CTA per right-hand side,
//      column-oriented back substitution                  (srqr_solve_kernel)
//   5. g2 ~= |alpha| / sqrt(d) max_i ||Y(i, :)||  (srqr_g2_kernel)
#pragma once
#include "common.cuh"
#include "philox.cuh"

namespace rq {

constexpr uint32_t SRQR_STREAM = 7;
constexpr int SRQR_THREADS = 256;

// argmax of the squared column norms of the l x nt sample (ld ldb), ties ->
// lowest column; one CTA.  out: *iota.
__global__ void __launch_bounds__(SRQR_THREADS) srqr_pick_kernel(const double *B, int64_t ldb, int l, int64_t nt,
                                                                 int *iota) {
    __shared__ double sv[SRQR_THREADS / 32];
    __shared__ int64_t sc[SRQR_THREADS / 32];
    double bv = -1.0;
    int64_t bc = INT64_MAX;
    for (int64_t c = threadIdx.x; c < nt; c += SRQR_THREADS) {
        double s = 0.0;
        for (int t = 0; t < l; ++t) s += B[t + c * ldb] * B[t + c * ldb];
        if (s > bv || (s == bv && c < bc)) { bv = s; bc = c; }
    }
    for (int o = 16; o > 0; o >>= 1) {
        const double ov = __shfl_xor_sync(0xffffffffu, bv, o);
        const int64_t oc = __shfl_xor_sync(0xffffffffu, bc, o);
        if (ov > bv || (ov == bv && oc < bc)) { bv = ov; bc = oc; }
    }
    if ((threadIdx.x & 31) == 0) { sv[threadIdx.x >> 5] = bv; sc[threadIdx.x >> 5] = bc; }
    __syncthreads();
    if (threadIdx.x == 0) {
        for (int w = 1; w < SRQR_THREADS / 32; ++w)
            if (sv[w] > sv[0] || (sv[w] == sv[0] && sc[w] < sc[0])) { sv[0] = sv[w]; sc[0] = sc[w]; }
        *iota = (int)sc[0];
    }
}

// swap lists for positions k <-> k + iota (relative to column k), for the S3 kernels
__global__ void srqr_swaplist_kernel(const int *iota, int64_t *dst, int64_t *src, int *np) {
    const int64_t q = *iota;
    if (q == 0) { *np = 0; return; }
    dst[0] = 0; src[0] = q;
    dst[1] = q; src[1] = 0;
    *np = 2;
}

// column norms of A(k:m, k:n): out[0] = max (as ordered bits of a non-negative
// double), out[1] = norm of column k.  Warp per column.
__global__ void srqr_norms_kernel(const double *A /* &A[k + k lda] */, int64_t lda, int64_t rows, int64_t cols,
                                  unsigned long long *maxbits, double *alpha) {
    const int warp = (blockIdx.x * blockDim.x + threadIdx.x) >> 5, lane = threadIdx.x & 31;
    const int nw = (gridDim.x * blockDim.x) >> 5;
    for (int64_t c = warp; c < cols; c += nw) {
        double s = 0.0;
        for (int64_t r = lane; r < rows; r += 32) s += A[r + c * lda] * A[r + c * lda];
        s = warp_sum(s);
        const double nrm = sqrt(s);
        if (lane == 0) {
            atomicMax(maxbits, (unsigned long long)__double_as_longlong(nrm));
            if (c == 0) *alpha = nrm;
        }
    }
}

// R-hat y = omega for right-hand side blockIdx.x (omega_j = N(0,1) entry
// (blockIdx.x, j) of (seed, stream 7)); R-hat(0:k, 0:k) = triu A(0:k, 0:k),
// R-hat(0:k, k) = A(0:k, k), R-hat(k, k) = *alpha.  Column-oriented back
// substitution with the right-hand side in shared memory (thread t updates
// rows t, t + 256, ... with column j of R-hat read from A).  Y: (k+1) x d.
__global__ void __launch_bounds__(SRQR_THREADS) srqr_solve_kernel(const double *A, int64_t lda, int64_t k,
                                                                  const double *alpha, uint64_t seed, double *Y) {
    extern __shared__ double sb[];  // k + 1
    const int rhs = blockIdx.x, tid = threadIdx.x;
    for (int64_t j = tid; j <= k; j += SRQR_THREADS) {
        const double2 z = normal_pair(seed, SRQR_STREAM, rhs >> 1, j);
        sb[j] = (rhs & 1) ? z.y : z.x;
    }
    __syncthreads();
    const double al = *alpha;
    for (int64_t j = k; j >= 0; --j) {
        const double rjj = (j == k) ? al : A[j + j * lda];
        const double yj = sb[j] / rjj;
        __syncthreads();  // every thread has read sb[j]
        if (tid == 0) sb[j] = yj;
        for (int64_t r = tid; r < j; r += SRQR_THREADS) sb[r] -= yj * A[r + j * lda];
        __syncthreads();
    }
    for (int64_t j = tid; j <= k; j += SRQR_THREADS) Y[j + (int64_t)rhs * (k + 1)] = sb[j];
}

// g2 estimate and the tau caps: out = {g1, g2_est, |alpha|, tau cap (Eq. 10),
// tau-hat cap (Eq. 12), iota}
__global__ void __launch_bounds__(SRQR_THREADS) srqr_g2_kernel(const double *Y, int64_t k, int d,
                                                               const unsigned long long *maxbits, const double *alpha,
                                                               const int *iota, int64_t n, double *out) {
    __shared__ double sm[SRQR_THREADS / 32];
    double mx = 0.0;
    for (int64_t i = threadIdx.x; i <= k; i += SRQR_THREADS) {
        double s = 0.0;
        for (int q = 0; q < d; ++q) s += Y[i + (int64_t)q * (k + 1)] * Y[i + (int64_t)q * (k + 1)];
        mx = fmax(mx, s);
    }
    for (int o = 16; o > 0; o >>= 1) mx = fmax(mx, __shfl_xor_sync(0xffffffffu, mx, o));
    if ((threadIdx.x & 31) == 0) sm[threadIdx.x >> 5] = mx;
    __syncthreads();
    if (threadIdx.x == 0) {
        for (int w = 1; w < SRQR_THREADS / 32; ++w) mx = fmax(mx, sm[w]);
        mx = fmax(mx, sm[0]);
        const double al = *alpha;
        const double cmax = __longlong_as_double((long long)*maxbits);
        const double g1 = cmax / al;
        const double g2 = al / sqrt((double)d) * sqrt(mx);
        out[0] = g1;
        out[1] = g2;
        out[2] = al;
        out[3] = g1 * g2 * sqrt((double)(k + 1) * (double)(n - k));
        out[4] = g1 * g2 * sqrt((double)k * (double)(n - k));
        out[5] = (double)*iota;
    }
}

}  // namespace rq
