// tri.cuh -- the two small b x b triangular computations of a panel, done
// by block-recursive doubling so that no thread runs a b^2-long serial chain:
//
//  block 0: compact-WY T (PDLARFT) from Y = strict_upper(V^T V) and tau:
//     base 8x8 blocks by the column recurrence T(0:j,j) = -tau_j T(0:j,0:j) y_j,
//     then merges  T = [T1, -T1 Y12 T2; 0, T2]  for block sizes 8, 16, 32, 64.
//     Written negated (Tneg = -T) for the W2 = -T^T W contraction.
//  block 1: Omega-hat11 = R-hat11 R11^{-1} (Eq. (4), reading
//     R-G20): R11^{-1} by the same doubling (inverse 8x8 blocks, then
//     B <- -A^{-1} B D^{-1}), then the upper-triangular product, written
//     TRANSPOSED (omhat[c + r bbpad] = Omega-hat11(r, c)) for the DMMA product
//     Omega-hat11 R12 of the sample update.
//
// One CTA each, run on a side stream concurrently with W = V^T A22 (neither
// result is needed before W2 = -T^T W / the sample update).  Entries beyond
// the panel's effective width are zero (tau = 0, identity blocks).
#pragma once
#include "common.cuh"

namespace rq {

constexpr int TRI_THREADS = 256;

// C(s x s) = A(s x s, upper) * B(s x s, upper)  (result upper); all in smem, ld given.
RQ_DEV void tri_mul_uu(const double *A, int lda, const double *B, int ldb, double *C, int ldc, int s, double alpha) {
    for (int e = threadIdx.x; e < s * s; e += blockDim.x) {
        const int r = e % s, c = e / s;
        double acc = 0.0;
        if (r <= c)
            for (int q = r; q <= c; ++q) acc += A[r + q * lda] * B[q + c * ldb];
        C[r + c * ldc] = alpha * acc;
    }
}

// C(s x s) = A(s x s, upper) * B(s x s, full); then D = C * E(upper) scaled.
RQ_DEV void tri_mul_uf(const double *A, int lda, const double *B, int ldb, double *C, int ldc, int s) {
    for (int e = threadIdx.x; e < s * s; e += blockDim.x) {
        const int r = e % s, c = e / s;
        double acc = 0.0;
        for (int q = r; q < s; ++q) acc += A[r + q * lda] * B[q + c * ldb];
        C[r + c * ldc] = acc;
    }
}
RQ_DEV void tri_mul_fu(const double *A, int lda, const double *B, int ldb, double *C, int ldc, int s, double alpha) {
    for (int e = threadIdx.x; e < s * s; e += blockDim.x) {
        const int r = e % s, c = e / s;
        double acc = 0.0;
        for (int q = 0; q <= c; ++q) acc += A[r + q * lda] * B[q + c * ldb];
        C[r + c * ldc] = alpha * acc;
    }
}

// Shared memory of tri_kernel: the nb x nb working triangle with an odd
// leading dimension (nb + 1: row- and column-wise walks are both free of bank
// conflicts), whose strictly lower part holds the second operand transposed
// (Y, or R-hat11), then (nb/2)^2 doubles of scratch and nb diagonal entries.
inline size_t tri_smem_bytes(int nb) {
    return ((size_t)nb * (nb + 1) + (size_t)(nb / 2) * (nb / 2) + (size_t)nb) * sizeof(double);
}

// nb = power of two multiple of 8, >= bb.  Every operand is staged in shared
// memory once (coalesced); no serial chain waits on global memory.
__global__ void __launch_bounds__(TRI_THREADS) tri_kernel(const double *ybuf /* bbpad x bbpad */, const double *tau,
                                                          const double *rhat11 /* bbpad x bbpad */,
                                                          const double *R11 /* &A[i+i lda] */, int64_t lda, int bb,
                                                          int bbpad, int nb, const int *bb_eff, double *tneg,
                                                          double *omhat, int do_omhat, const int *t_ready) {
    extern __shared__ __align__(16) double tsm[];
    const int ld = nb + 1;
    double *M = tsm;                       // nb x nb, ld nb + 1: upper = result, strict lower = operand^T
    double *tmp = tsm + (size_t)nb * ld;   // (nb/2) x (nb/2)
    double *dg = tmp + (nb / 2) * (nb / 2); // nb: diagonal of the staged operand
    const int bbe = *bb_eff;
    const int tid = threadIdx.x;
    if (blockIdx.x == 0) {
        // ---------------- T ----------------
        if (t_ready && *t_ready == 0) return;  // written by the CholeskyQR2 reconstruction
        // upper: 0; strict lower M(r, c) (r > c) = Y(c, r) = v_c^T v_r (c < r < bbe)
        for (int e = tid; e < nb * nb; e += blockDim.x) {
            const int c = e % nb, r = e / nb;  // consecutive threads: consecutive c (coalesced ybuf column r)
            M[r + c * ld] = (r > c && r < bbe) ? ybuf[c + (int64_t)r * bbpad] : 0.0;
        }
        for (int j = tid; j < nb; j += blockDim.x) dg[j] = (j < bbe) ? tau[j] : 0.0;
        __syncthreads();
        // base: each thread owns one 8x8 diagonal block, column recurrence
        // T(r, j) = -tau_j sum_{r <= c < j} T(r, c) Y(c, j)
        if (tid < nb / 8) {
            const int k0 = tid * 8;
            for (int j = k0; j < k0 + 8; ++j) {
                if (j >= bbe) continue;  // tau = 0 beyond the effective width: zero column
                const double tj = dg[j];
                for (int r = k0; r < j; ++r) {
                    double acc = 0.0;
                    for (int c = r; c < j; ++c) acc += M[r + c * ld] * M[j + c * ld];
                    M[r + j * ld] = -tj * acc;
                }
                M[j + j * ld] = tj;
            }
        }
        __syncthreads();
        for (int s = 8; s < nb; s *= 2) {
            for (int k = 0; k < nb; k += 2 * s) {
                // tmp = Y12 * T2 ; T12 = -T1 * tmp  (Y12(r, q) = M(k + s + q, k + r))
                for (int e = tid; e < s * s; e += blockDim.x) {
                    const int r = e % s, c = e / s;
                    double acc = 0.0;
                    for (int q = 0; q <= c; ++q) acc += M[(k + s + q) + (k + r) * ld] * M[(k + s + q) + (k + s + c) * ld];
                    tmp[r + c * (nb / 2)] = acc;
                }
                __syncthreads();
                tri_mul_uf(M + k + k * ld, ld, tmp, nb / 2, M + k + (k + s) * ld, ld, s);
                __syncthreads();
            }
            // negate T12 blocks of this level
            for (int k = 0; k < nb; k += 2 * s)
                for (int e = tid; e < s * s; e += blockDim.x) {
                    const int r = e % s, c = e / s;
                    M[(k + r) + (k + s + c) * ld] = -M[(k + r) + (k + s + c) * ld];
                }
            __syncthreads();
        }
        for (int e = tid; e < bbpad * bbpad; e += blockDim.x) {
            const int r = e % bbpad, c = e / bbpad;
            tneg[e] = (r <= c && c < nb) ? -M[r + c * ld] : 0.0;
        }
    } else {
        // ---------------- Omega-hat11 = R-hat11 R11^{-1} ----------------
        if (!do_omhat || bbe != bb) return;
        // upper: R11 (identity padding); strict lower M(r, c) (r > c) = R-hat11(c, r); dg = diag(R-hat11)
        for (int e = tid; e < nb * nb; e += blockDim.x) {
            const int r = e % nb, c = e / nb;
            if (r > c) continue;  // the strict lower part is the next loop's
            double v = 0.0;
            if (r < bb && c < bb) v = R11[r + (int64_t)c * lda];
            else if (r == c) v = 1.0;
            M[r + c * ld] = v;
        }
        for (int e = tid; e < nb * nb; e += blockDim.x) {
            const int c = e % nb, r = e / nb;  // R-hat11(c, r), c < r: coalesced column r
            if (r > c) M[r + c * ld] = (r < bb) ? rhat11[c + (int64_t)r * bbpad] : 0.0;
        }
        for (int j = tid; j < nb; j += blockDim.x) dg[j] = (j < bb) ? rhat11[j + (int64_t)j * bbpad] : 0.0;
        __syncthreads();
        // base: invert 8x8 diagonal blocks in place (thread per block column-by-column)
        if (tid < nb / 8) {
            const int k0 = tid * 8;
            double inv[8][8];
            for (int c = 0; c < 8; ++c)
                for (int r = 0; r < 8; ++r) inv[r][c] = 0.0;
            for (int c = 0; c < 8; ++c) {
                // solve U x = e_c (back substitution), U = M[k0.., k0..]
                for (int r = c; r >= 0; --r) {
                    double s = (r == c) ? 1.0 : 0.0;
                    for (int q = r + 1; q <= c; ++q) s -= M[(k0 + r) + (k0 + q) * ld] * inv[q][c];
                    inv[r][c] = s / M[(k0 + r) + (k0 + r) * ld];
                }
            }
            for (int c = 0; c < 8; ++c)
                for (int r = 0; r <= c; ++r) M[(k0 + r) + (k0 + c) * ld] = inv[r][c];
        }
        __syncthreads();
        for (int s = 8; s < nb; s *= 2) {
            for (int k = 0; k < nb; k += 2 * s) {
                // B <- -A^{-1} B D^{-1}:  tmp = A^{-1} B ; B = -tmp D^{-1}
                tri_mul_uf(M + k + k * ld, ld, M + k + (k + s) * ld, ld, tmp, nb / 2, s);
                __syncthreads();
                tri_mul_fu(tmp, nb / 2, M + (k + s) + (k + s) * ld, ld, M + k + (k + s) * ld, ld, s, -1.0);
                __syncthreads();
            }
        }
        // Omega-hat = R-hat11 * R11^{-1} (upper x upper)
        for (int e = tid; e < bbpad * bbpad; e += blockDim.x) {
            const int r = e % bbpad, c = e / bbpad;
            double acc = 0.0;
            if (r <= c && c < bb) {
                acc = dg[r] * M[r + c * ld];
                for (int q = r + 1; q <= c; ++q) acc += M[q + r * ld] * M[q + c * ld];
            }
            omhat[c + r * bbpad] = acc;  // stored transposed: the K-contiguous X of C = X^T R12
        }
    }
}

}  // namespace rq
