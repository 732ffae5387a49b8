// lowrank.cuh -- low-rank outputs of the partial QRCP (
// SURVEY.md §8(f) N4): the explicit Q1 (first k columns of
// Q = H_1 ... H_k) and the CX coefficient matrix X = C^+ A with
// C = A Pi(:, 0:k) the first k pivot columns.
//
// Q1: X = [I_k; 0], then for every panel from the last to the first
// X(i:m, i:k) <- (I - V T V^T) X(i:m, i:k) with the panel's V (from the
// factored A) and T (from V^T V and tau, tri.cuh) -- the trailing-update
// contractions with the roles of the operands swapped.
// CX: C = Q1 R11 (Householder QR of the pivot columns), so
// X Pi = R11^{-1} Q1^T A Pi = [I, R11^{-1} R12]; Z = R11^{-1} R12 by a blocked
// back substitution (64-row blocks from the bottom: a DMMA contraction with
// the already solved rows, then a 64 x 64 triangular solve per column).
#pragma once
#include "common.cuh"

namespace rq {

__global__ void lr_set_int_kernel(int *p, int v) { *p = v; }

// X (rows x cols, ldx) = [I; 0]
__global__ void lr_eye_kernel(double *X, int64_t ldx, int64_t rows, int64_t cols) {
    const int64_t total = rows * cols;
    for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < total; e += (int64_t)gridDim.x * blockDim.x) {
        const int64_t r = e % rows, c = e / rows;
        X[r + c * ldx] = (r == c) ? 1.0 : 0.0;
    }
}

// explicit V (mp x bbpad, ld ldv: unit diagonal, zeros above and beyond bb)
// and V^T (bbpad x mp) of the panel whose top-left is P (ld lda)
__global__ void lr_extract_v_kernel(const double *P, int64_t lda, int64_t mp, int bb, int bbpad, double *vfull,
                                    int64_t ldv, double *vt) {
    const int64_t total = mp * bbpad;
    for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < total; e += (int64_t)gridDim.x * blockDim.x) {
        const int64_t r = e % mp;
        const int c = (int)(e / mp);
        double v = 0.0;
        if (c < bb) v = (r > c) ? P[r + (int64_t)c * lda] : (r == c ? 1.0 : 0.0);
        vfull[r + (int64_t)c * ldv] = v;
        vt[c + r * bbpad] = v;
    }
}

// out = in^T (n x n, ld n)
__global__ void lr_transpose_kernel(const double *in, int n, double *out) {
    for (int e = blockIdx.x * blockDim.x + threadIdx.x; e < n * n; e += gridDim.x * blockDim.x) {
        const int r = e % n, c = e / n;
        out[c + r * n] = in[e];
    }
}

// RT (k x k, ld k) = R11^T: lower triangular, R11 = triu(A(0:k, 0:k))
__global__ void lr_r11t_kernel(const double *A, int64_t lda, int64_t k, double *RT) {
    const int64_t total = k * k;
    for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < total; e += (int64_t)gridDim.x * blockDim.x) {
        const int64_t r = e % k, c = e / k;  // RT(r, c) = R11(c, r)
        RT[r + c * k] = (r >= c) ? A[c + r * lda] : 0.0;
    }
}

// Z(r0:r0+bs, c) = R11(r0:r0+bs, r0:r0+bs)^{-1} (R12(r0:r0+bs, c) - C(0:bs, c))
// for c < n2; thread per column, the bs x bs diagonal block in shared memory.
// R12(:, c) = A(0:k, k + c); C may be null (the bottom block).
__global__ void lr_block_solve_kernel(const double *A, int64_t lda, int64_t k, int64_t n2, int64_t r0, int bs,
                                      const double *C, int64_t ldc, double *Z, int64_t ldz) {
    __shared__ double Rb[64 * 64];
    for (int e = threadIdx.x; e < bs * bs; e += blockDim.x) {
        const int r = e % bs, c = e / bs;
        Rb[r + c * 64] = (r <= c) ? A[(r0 + r) + (r0 + c) * lda] : 0.0;
    }
    __syncthreads();
    const int64_t col = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (col >= n2) return;
    double y[64];
#pragma unroll
    for (int r = 0; r < 64; ++r)
        y[r] = (r < bs) ? A[(r0 + r) + (k + col) * lda] - (C ? C[r + col * ldc] : 0.0) : 0.0;
#pragma unroll
    for (int r = 63; r >= 0; --r) {
        if (r < bs) {
            double s = y[r];
#pragma unroll
            for (int q = r + 1; q < 64; ++q)
                if (q < bs) s -= Rb[r + q * 64] * y[q];
            y[r] = s / Rb[r + r * 64];
        }
    }
#pragma unroll
    for (int r = 0; r < 64; ++r)
        if (r < bs) Z[(r0 + r) + col * ldz] = y[r];
}

// X (k x n, ldx) in the original column order: X(:, jpvt[j]) = e_j (j < k),
// = Z(:, j - k) (j >= k)
__global__ void lr_cx_scatter_kernel(const double *Z, int64_t ldz, const int64_t *jpvt, int64_t k, int64_t n,
                                     double *X, int64_t ldx) {
    const int64_t total = k * n;
    for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < total; e += (int64_t)gridDim.x * blockDim.x) {
        const int64_t r = e % k, j = e / k;
        const double v = (j < k) ? (r == j ? 1.0 : 0.0) : Z[r + (j - k) * ldz];
        X[r + jpvt[j] * ldx] = v;
    }
}

}  // namespace rq
